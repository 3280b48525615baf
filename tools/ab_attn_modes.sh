#!/bin/bash
# Attention backward microbenchmark over {serial, concurrent dQ} x {LPT, head-major grid}, twice each.
set -u
P=${1:-r02q2}
O=gpurun_out
for k in 1 2; do
for conc in 1 0; do
for lpt in 1 0; do
  unset MALLEUS_ATTN_BWD_SERIAL MALLEUS_ATTN_GRID_HEADMAJOR
  [ $conc = 0 ] && export MALLEUS_ATTN_BWD_SERIAL=1
  [ $lpt = 0 ] && export MALLEUS_ATTN_GRID_HEADMAJOR=1
  echo "== conc=$conc lpt=$lpt run $k"
  timeout 300 python tools/attn_bench.py 2>&1 | grep "nb="
done
done
done
