#!/bin/bash
# ncu --set full of the fused variation + mask kernel at C4 (one launch), optionally with diagnostic bits; raw + source pages as csv
TAG=${1:-vary}; DIAG=${2:-0}
GAPA_NVCC_EXTRA="-DGAPA_VARY_DIAG=$DIAG ${EXTRA:-}" python paper_2412_20980_b200/build.py --force > /dev/null 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_pc_bitmask_vary -c 1 -o gpurun_out/${TAG} -f \
    python tools/probe_gen.py c4 > /dev/null 2>&1
ncu -i gpurun_out/${TAG}.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>/dev/null
ncu -i gpurun_out/${TAG}.ncu-rep --page source --csv > gpurun_out/${TAG}_source.csv 2>/dev/null
rm -f gpurun_out/${TAG}.ncu-rep
python paper_2412_20980_b200/build.py --force > /dev/null 2>&1
