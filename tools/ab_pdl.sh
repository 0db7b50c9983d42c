#!/bin/bash
# A/B on the GPU box: programmatic dependent launch of every kernel (GAPA_PDL=0/1) — bench step and library loop per workload
for w in ${WORKLOADS:-c1 c3 n1e4 n1e5 c4}; do
  for v in 0 1; do
    echo "== $w GAPA_PDL=$v"
    steps=30; [ $w = c1 ] && steps=200; [ $w = c3 ] && steps=200
    for i in 1 2; do GAPA_PDL=$v python bench.py --workload $w --steps $steps --warmup 10 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('step %.5f ms  %.0f gen/s   eval %.5f ms   library loop %.0f gen/s   e2e %.4g' % (d['ms_per_step'], d['generations_per_sec'], d['fitness_eval_ms_per_step'], d['library_loop']['generations_per_sec'], d['e2e']['value']))"; done
  done
done
