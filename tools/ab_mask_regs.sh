#!/bin/bash
# A/B on the GPU box: register cap of the persistent plain mask kernel (room for the clearing kernel beside it on an SM)
for v in ${VARIANTS:-0 56 48 40}; do
  echo "== GAPA_MASK_MAXREG=$v"
  GAPA_NVCC_EXTRA="-DGAPA_MASK_MAXREG=$v" python paper_2412_20980_b200/build.py --force > /dev/null 2>&1 || { echo build failed; continue; }
  for w in c4 n1e5; do for i in 1 2; do python tools/probe_eval.py $w 2>&1 | tail -1 | cut -c1-90; done; done
done
python paper_2412_20980_b200/build.py --force > /dev/null 2>&1
