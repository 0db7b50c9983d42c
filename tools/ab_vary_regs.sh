#!/bin/bash
# A/B on the GPU box: register cap of the fused variation kernel (-DGAPA_VARY_MAXREG=n; 0 = __launch_bounds__ only, 64 registers).
# With 56 registers two clearing CTAs fit beside it on an SM again and the clear runs underneath it instead of beside the transpose.
for v in ${VARIANTS:-0 56 48}; do
  echo "== GAPA_VARY_MAXREG=$v"
  GAPA_NVCC_EXTRA="-DGAPA_VARY_MAXREG=$v" python paper_2412_20980_b200/build.py --force > /dev/null 2>&1 || { echo build failed; continue; }
  for w in c4 n1e5; do for i in 1 2; do python tools/probe_gen_kernels.py $w 2>&1 | tail -1; done; done
done
python paper_2412_20980_b200/build.py --force > /dev/null 2>&1
