#!/bin/bash
for w in c4 n1e5 n1e4 c3; do
  for v in 0 592 2368; do
    echo "== $w GAPA_PDL_MAX_CTAS=$v"
    steps=30; [ $w = c3 ] && steps=200
    GAPA_PDL_MAX_CTAS=$v python bench.py --workload $w --steps $steps --warmup 10 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('step %.5f ms  eval %.5f ms   library loop %.0f gen/s' % (d['ms_per_step'], d['fitness_eval_ms_per_step'], d['library_loop']['generations_per_sec']))"
  done
done
