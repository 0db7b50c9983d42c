#!/bin/bash
# Generic compile-time A/B on the GPU box: each argument is a set of nvcc defines; per variant the per-kernel time of a
# generation (tools/probe_gen_kernels.py, WORKLOAD, default c4), repeated REPS times; the default build is restored at the end.
for v in "$@"; do
  echo "== [$v]"
  GAPA_NVCC_EXTRA="$v" python paper_2412_20980_b200/build.py --force > /dev/null 2>&1 || { echo build failed; continue; }
  for r in $(seq ${REPS:-2}); do python tools/probe_gen_kernels.py ${WORKLOAD:-c4} 2>&1 | tail -1; done
done
python paper_2412_20980_b200/build.py --force > /dev/null 2>&1
