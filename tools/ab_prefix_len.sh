#!/bin/bash
# A/B of the prefix length and the sweep interleave (runtime knobs) across sizes
CONFIGS=${CONFIGS:-"c4:4096 c4:1024 c4:16384 n1e5:4096"}
KNOBS=${KNOBS:-"8:32768 8:65536 8:131072 16:32768 16:65536"}
for rep in 1 2; do for kn in $KNOBS; do for cfg in $CONFIGS; do
  GAPA_PC_INTERLEAVE=${kn%:*} GAPA_PC_PREFIX=${kn#*:} timeout 300 python bench.py --workload ${cfg%:*} --pop ${cfg#*:} --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.readlines()[-1]); print('il:prefix=$kn', '$cfg', round(d['ms_per_step'],4), round(d['fitness_eval_ms_per_step'],4))"
done; done; done
