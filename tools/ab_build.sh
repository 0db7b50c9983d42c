#!/bin/bash
# A/B compile-time variants on the GPU box (nvcc is in the image): rebuild, probe, restore.
for v in "$@"; do
  echo "== $v"
  GAPA_NVCC_EXTRA="$v" python paper_2412_20980_b200/build.py --force > /dev/null 2>&1 || { echo build failed; continue; }
  python tools/probe_pc.py 1e6 4096 2>&1 | grep -E "iter [34]"
done
