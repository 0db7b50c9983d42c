#!/bin/bash
# A/B of the persistent fused variation + mask kernel on the GPU box (C4 generation; also n = 1e5 / 1e4 where the CTAs are small):
# GAPA_PC_VARY_WAVES = 1 (persistent: one CTA per resident slot walks its rows) vs a large value (one row per CTA).
for w in c4 n1e5 n1e4; do
  for v in 1 2 100000; do
    echo "== $w GAPA_PC_VARY_WAVES=$v"
    for i in 1 2; do GAPA_PC_VARY_WAVES=$v python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('step %.4f ms  eval %.4f ms  loop %.1f gen/s' % (d['ms_per_step'], d['fitness_eval_ms_per_step'], d['library_loop']['generations_per_sec']))"; done
  done
done
