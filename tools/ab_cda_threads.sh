#!/bin/bash
# A/B of the CDA kernel's CTA size on the GPU box (nvcc is in the image): C2 batch of 100 and a larger graph
for v in "-DGAPA_CDA_THREADS=1024" "-DGAPA_CDA_THREADS=512" "-DGAPA_CDA_THREADS=256" "-DGAPA_CDA_THREADS=128" "-DGAPA_CDA_THREADS=512 -DGAPA_CDA_GROUP=4" "-DGAPA_CDA_THREADS=256 -DGAPA_CDA_GROUP=4"; do
  echo "== $v"
  GAPA_NVCC_EXTRA="$v" python paper_2412_20980_b200/build.py --force > /dev/null 2>&1 || { echo build failed; continue; }
  python tools/probe_cda.py 10 500 100 2>&1 | grep "rows=" | tail -1
  python tools/probe_cda.py 10 500 296 2>&1 | grep "rows=" | tail -1
  python tools/probe_cda.py 20 1000 20 2>&1 | grep "rows=" | tail -1
done
python paper_2412_20980_b200/build.py --force > /dev/null 2>&1
