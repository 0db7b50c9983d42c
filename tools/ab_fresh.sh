#!/bin/bash
# A/B on the GPU box: the first sweep skips loading records known to be clear (GAPA_PC_FRESH_SKIP) — evaluation and generation
for w in c4 n1e5 n1e4; do
  for v in 0 1; do
    echo "== $w GAPA_PC_FRESH_SKIP=$v"
    GAPA_PC_FRESH_SKIP=$v python tools/probe_gen_kernels.py $w 2>&1 | tail -1
    GAPA_PC_FRESH_SKIP=$v python tools/probe_eval.py $w 2>&1 | tail -1
  done
done
