#!/bin/bash
# Graph families other than Barabasi-Albert (tools/probe_pc_misc.py) through the bit-sliced pipeline (GAPA_PC_UF=0), the
# per-individual union-find (1) and the automatic, measured choice (-1)
for v in 0 1 -1; do
  echo "== GAPA_PC_UF=$v"
  GAPA_PC_UF=$v python tools/probe_pc_misc.py 2>&1 | grep "device"
done
