#!/bin/bash
# A/B of the lane schedule of the PC evaluation: individuals per lane x lanes in flight.
# Prints the bench step (one generation) and the pure evaluation time.  usage: tools/ab_lanes.sh [workload] [pop]
W=${1:-c4}; POP=${2:-0}
for cfg in "GAPA_PC_LANE_ROWS=1048576 GAPA_PC_LANE_STREAMS=1" "GAPA_PC_LANE_ROWS=2048 GAPA_PC_LANE_STREAMS=2" "GAPA_PC_LANE_ROWS=1024 GAPA_PC_LANE_STREAMS=2" \
           "GAPA_PC_LANE_ROWS=1024 GAPA_PC_LANE_STREAMS=3" "GAPA_PC_LANE_ROWS=1024 GAPA_PC_LANE_STREAMS=4" "GAPA_PC_LANE_ROWS=512 GAPA_PC_LANE_STREAMS=2" \
           "GAPA_PC_LANE_ROWS=512 GAPA_PC_LANE_STREAMS=3" "GAPA_PC_LANE_ROWS=512 GAPA_PC_LANE_STREAMS=4" "GAPA_PC_LANE_ROWS=256 GAPA_PC_LANE_STREAMS=4" \
           "GAPA_PC_LANE_ROWS=256 GAPA_PC_LANE_STREAMS=8" "GAPA_PC_LANE_ROWS=1024 GAPA_PC_LANE_STREAMS=2 GAPA_PC_SPEC_ROUNDS=0"; do
  echo "== $cfg"
  env $cfg python bench.py --workload $W --pop $POP --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    l=l.strip()
    if l.startswith('{'):
        d=json.loads(l); print('step %.3f ms  eval %.3f ms  vary+eval %.3f ms  launches %d  loop %.1f gen/s' % (d['ms_per_step'], d['fitness_eval_ms_per_step'], d['variation_plus_eval_ms_per_step'], d['gpu_launches'], d.get('library_loop',{}).get('generations_per_sec',0)))
    elif l: print(l[:300])
"
done
