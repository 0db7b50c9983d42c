#!/bin/bash
# A/B on the GPU box: L2 prefetch distance (in 256-vertex chunks) of the ordinary sweep's own-vertex data
for w in ${WORKLOADS:-c4 n1e5}; do
  for v in ${VARIANTS:-0 8 16 32 64 128 256}; do
    echo "== $w GAPA_PC_SWEEP_PREFETCH=$v"
    GAPA_PC_SWEEP_PREFETCH=$v python tools/probe_gen_kernels.py $w 2>&1 | tail -1
  done
done
