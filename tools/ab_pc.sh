#!/bin/bash
# A/B probe of the PC tuning knobs on C4 (device-side eval time only)
for cfg in "GAPA_PC_PREFIX=65536 GAPA_PC_INTERLEAVE=16" "GAPA_PC_PREFIX=49152 GAPA_PC_INTERLEAVE=16" "GAPA_PC_PREFIX=32768 GAPA_PC_INTERLEAVE=16" "GAPA_PC_PREFIX=65536 GAPA_PC_INTERLEAVE=12" "GAPA_PC_PREFIX=65536 GAPA_PC_INTERLEAVE=24" "GAPA_PC_PREFIX=98304 GAPA_PC_INTERLEAVE=16"; do
  echo "== $cfg"; env $cfg python tools/probe_pc.py ${1:-1e6} 4096 2>&1 | grep -E "iter [34]|oracle"
done
