#!/bin/bash
# A/B probe of the PC tuning knobs (device-side eval time only)
for cfg in "GAPA_PC_PREFIX_FIRST4=0" "GAPA_PC_PREFIX_FIRST4=1" "GAPA_PC_PREFIX_FIRST4=1 GAPA_PC_PREFIX=65536" "GAPA_PC_PREFIX_FIRST4=1 GAPA_PC_PREFIX=131072" "GAPA_PC_PREFIX_FIRST4=1 GAPA_PC_PREFIX=16384"; do
  echo "== $cfg"; env $cfg python tools/probe_pc.py ${1:-1e6} ${2:-4096} 2>&1 | grep -E "iter [34]|oracle"
done
