#!/bin/bash
# crossover between the per-individual small-graph kernel and the bit-sliced pipeline (device eval time)
for n in 1e3 3e3 1e4 1.6e4; do for pop in 64 256 1024 4096; do
  a=$(GAPA_PC_SMALL=1 python tools/probe_pc.py $n $pop 2>&1 | grep "iter 4" | sed 's/.*device \([0-9.]*\) ms.*/\1/')
  b=$(GAPA_PC_SMALL=0 python tools/probe_pc.py $n $pop 2>&1 | grep "iter 4" | sed 's/.*device \([0-9.]*\) ms.*/\1/')
  echo "n=$n pop=$pop small=$a ms  bitsliced=$b ms"
done; done
