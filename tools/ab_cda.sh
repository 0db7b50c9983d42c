#!/bin/bash
# A/B compile-time variants of the CDA patch thresholds on the GPU box (nvcc is in the image)
for v in "-DGAPA_CDA_SHORT=64" "-DGAPA_CDA_SHORT=128" "-DGAPA_CDA_SHORT=256" "-DGAPA_CDA_THREADLIST=12" "-DGAPA_CDA_THREADLIST=48" "-DGAPA_CDA_GROUP=4" "-DGAPA_CDA_GROUP=16 -DGAPA_CDA_SHORT=128" "-DGAPA_CDA_GROUP=32 -DGAPA_CDA_SHORT=256"; do
  echo "== $v"
  GAPA_NVCC_EXTRA="$v" python paper_2412_20980_b200/build.py --force > /dev/null 2>&1 || { echo build failed; continue; }
  python tools/probe_cda.py 10 500 100 2>&1 | grep "rows=" | tail -1
  python tools/probe_cda.py 20 1000 20 2>&1 | grep "rows=" | tail -1
done
