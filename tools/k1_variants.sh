#!/bin/bash
# ncu the K1 kernel in isolation for several CTA tilings (MBS_K1_TILE; 0 = balanced over resident CTAs)
for t in 0 4096 8192 16384 32768; do
  MBS_K1_TILE=$t ncu --set full --clock-control none -k regex:k_accum -c 6 -o gpurun_out/k1_tile$t \
      python tools/kbench.py --iters 1 > gpurun_out/k1_tile$t.txt 2>&1
done
