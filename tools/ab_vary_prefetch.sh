#!/bin/bash
# A/B of the L2 prefetch distance of the fused variation + mask kernel (passes ahead; 0 = off) — C4 generation on the GPU box.
# A second argument adds diagnostic bits (tools/ab_vary_diag.sh), e.g. 14 = loads + bitmap write-out only.
for v in ${VARIANTS:-0 1 2 3 4 6}; do
  echo "== GAPA_VARY_PREFETCH=$v DIAG=${DIAG:-0}"
  GAPA_NVCC_EXTRA="-DGAPA_VARY_PREFETCH=$v -DGAPA_VARY_DIAG=${DIAG:-0}" python paper_2412_20980_b200/build.py --force > /dev/null 2>&1 || { echo build failed; continue; }
  python tools/probe_gen_kernels.py ${WORKLOAD:-c4} 2>&1 | tail -1
done
python paper_2412_20980_b200/build.py --force > /dev/null 2>&1
