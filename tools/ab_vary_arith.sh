#!/bin/bash
# A/B of the hand-expanded integer arithmetic of the variation hash (variation.cuh) on the GPU box: C4 generation
for v in ${VARIANTS:-0 1 2 3 6}; do
  echo "== GAPA_VARY_ARITH=$v"
  GAPA_NVCC_EXTRA="-DGAPA_VARY_ARITH=$v" python paper_2412_20980_b200/build.py --force > /dev/null 2>&1 || { echo build failed; continue; }
  for i in 1 2; do python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('step %.4f ms  vary+eval %.4f ms' % (d['ms_per_step'], d['variation_plus_eval_ms_per_step']))"; done
done
python paper_2412_20980_b200/build.py --force > /dev/null 2>&1
python -m pytest tests/test_gpu_ga_ops.py tests/test_gpu_run.py -q -x 2>&1 | tail -2
