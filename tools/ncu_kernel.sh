#!/bin/bash
# ncu --set full of ONE kernel (regex) of one fitness evaluation / generation at a workload; raw + source pages as csv
# usage: bash tools/ncu_kernel.sh <tag> <kernel regex> [workload] [gen|eval]
TAG=$1; KRE=$2; W=${3:-c4}; WHAT=${4:-eval}
PROBE=tools/probe_eval.py; [ "$WHAT" = gen ] && PROBE=tools/probe_gen.py
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:$KRE -c 1 -o gpurun_out/${TAG} -f \
    python $PROBE $W > /dev/null 2>&1
ncu -i gpurun_out/${TAG}.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>/dev/null
ncu -i gpurun_out/${TAG}.ncu-rep --page source --csv > gpurun_out/${TAG}_source.csv 2>/dev/null
rm -f gpurun_out/${TAG}.ncu-rep
