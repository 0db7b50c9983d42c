#!/bin/bash
# A/B probe of the PC tuning knobs on C4 (device-side eval time only)
for cfg in "GAPA_PC_L1=1" "GAPA_PC_L1=0" "GAPA_PC_MASK_CHUNKS=2" "GAPA_PC_INTERLEAVE=4" "GAPA_PC_INTERLEAVE=16" "GAPA_PC_INTERLEAVE=64" "GAPA_PC_PREFIX=8192" "GAPA_PC_PREFIX=131072" "GAPA_PC_PREFIX=0"; do
  echo "== $cfg"; env $cfg python tools/probe_pc.py 1e6 4096 2>&1 | grep -E "iter [34]|oracle"
done
