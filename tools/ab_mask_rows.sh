#!/bin/bash
# A/B on the GPU box: persistent pipelined plain mask kernel (1) vs one CTA per row (0) — pure evaluation (tools/probe_eval.py)
for w in ${WORKLOADS:-c4 n1e5 n1e4}; do
  for v in 0 1; do
    echo "== $w GAPA_PC_MASK_ROWS=$v"
    for i in 1 2; do GAPA_PC_MASK_ROWS=$v python tools/probe_eval.py $w 2>&1 | tail -1; done
  done
done
