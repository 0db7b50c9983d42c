#!/bin/bash
# What bounds the fused variation + mask kernel?  Timing-only variants (results are wrong): GAPA_VARY_DIAG bits
# 1 = no parent loads, 2 = no bitmap marks, 4 = no child stores, 8 = no hashing.  C4 generation on the GPU box.
for v in ${VARIANTS:-0 1 2 4 8 3 7 9 14}; do
  echo "== GAPA_VARY_DIAG=$v"
  GAPA_NVCC_EXTRA="-DGAPA_VARY_DIAG=$v" python paper_2412_20980_b200/build.py --force > /dev/null 2>&1 || { echo build failed; continue; }
  python tools/probe_gen_kernels.py c4 2>&1 | tail -3
done
python paper_2412_20980_b200/build.py --force > /dev/null 2>&1
