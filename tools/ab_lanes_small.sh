#!/bin/bash
# A/B on the GPU box: lane size at population 16,384 on the small graphs (one lane vs lanes of 4096 / 8192 rows)
for w in n1e4 n1e5; do
  for v in 4096 8192 16384; do
    echo "== $w pop 16384 GAPA_PC_LANE_ROWS=$v"
    GAPA_PC_LANE_ROWS=$v python bench.py --workload $w --pop 16384 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('step %.4f ms  eval %.4f ms  loop %.1f gen/s  e2e %.3g' % (d['ms_per_step'], d['fitness_eval_ms_per_step'], d['library_loop']['generations_per_sec'], d['e2e']['value']))"
  done
done
