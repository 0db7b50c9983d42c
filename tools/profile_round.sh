#!/bin/bash
# The ncu passes behind profiles/ for one round (run on the B200 box under gpurun; tag = file prefix, e.g. r02a):
#   1. launch list of `bench.py` (C4 generation loop)           -> gpurun_out/<tag>_launches_c4.csv
#   2. launch lists of ONE fitness evaluation per workload with DRAM bytes (tools/probe_eval.py brackets it)
#                                                                -> gpurun_out/<tag>_eval_<workload>.csv
#   3. --set full of the main kernels at C4                      -> gpurun_out/<tag>_full_c4.ncu-rep + raw csv
# then, back in the repo:  python tools/ncu_traffic.py gpurun_out/<tag>_eval_c4.csv c4 profiles/<tag>_eval_c4.csv   (etc.)
TAG=${1:-r02a}
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors.sum
ncu --metrics $M --clock-control none -s 40 -c 60 --csv --log-file gpurun_out/${TAG}_launches_c4.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
for w in c4 n1e5 c1 c2 c3; do
  ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file gpurun_out/${TAG}_eval_${w}.csv \
      python tools/probe_eval.py $w > gpurun_out/${TAG}_eval_${w}.txt 2>&1
done
ncu --profile-from-start off --set full --clock-control none --import-source on -o gpurun_out/${TAG}_full_c4 -f \
    python tools/probe_gen.py c4 > /dev/null 2>&1
ncu -i gpurun_out/${TAG}_full_c4.ncu-rep --page raw --csv > gpurun_out/${TAG}_full_c4_raw.csv 2>/dev/null
rm -f gpurun_out/${TAG}_full_c4.ncu-rep   # large; the raw csv carries every metric of every launch
ls -la gpurun_out/${TAG}_*
