#!/bin/bash
# A/B of the prefix kernel's cluster size (GAPA_PC_PREFIX_CLUSTER: 0 = by super-group count; 1, 2, 4, 8 = fixed)
CLUSTERS=${CLUSTERS:-"0 8"}
CONFIGS=${CONFIGS:-"n1e4:8192 n1e4:16384 n1e5:16384 c4:4096 c4:8192 c4:16384"}
for rep in 1 2; do for c in $CLUSTERS; do for cfg in $CONFIGS; do
  GAPA_PC_PREFIX_CLUSTER=$c python bench.py --workload ${cfg%:*} --pop ${cfg#*:} --steps 20 --warmup 4 --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.readlines()[-1]); print('cluster=$c', '$cfg', round(d['ms_per_step'],4), round(d['fitness_eval_ms_per_step'],4))"
done; done; done
