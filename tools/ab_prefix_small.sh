#!/bin/bash
# prefix-closure knobs on small graphs (n = 1e4): prefix length, first-four-neighbours passes, cluster size
run() { python bench.py --workload n1e4 --pop $POP --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.readlines()[-1]); print('$1', 'pop=$POP', round(d['ms_per_step'],4), round(d['fitness_eval_ms_per_step'],4))"; }
for POP in 4096 16384; do
  run default
  for p in 0 1024 4096; do GAPA_PC_PREFIX=$p run prefix=$p; done
  GAPA_PC_PREFIX_FIRST4=0 run first4=0
  for c in 1 2 8; do GAPA_PC_PREFIX_CLUSTER=$c run cluster=$c; done
done
