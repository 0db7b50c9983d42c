#!/bin/bash
# A/B of the hand-expanded integer arithmetic of the variation hash (variation.cuh: GAPA_VARY_ARITH bits) on the GPU box:
# per-kernel time of a C4 generation (tools/probe_gen_kernels.py), then the operator / run tests on the default build.
for v in ${VARIANTS:-2 10 18 34 50 58}; do
  echo "== GAPA_VARY_ARITH=$v"
  GAPA_NVCC_EXTRA="-DGAPA_VARY_ARITH=$v" python paper_2412_20980_b200/build.py --force > /dev/null 2>&1 || { echo build failed; continue; }
  python tools/probe_gen_kernels.py ${WORKLOAD:-c4} 2>&1 | tail -1
  if [ -n "$TESTS" ]; then python -m pytest tests/test_gpu_ga_ops.py tests/test_gpu_run.py -q -x 2>&1 | tail -1; fi
done
python paper_2412_20980_b200/build.py --force > /dev/null 2>&1
