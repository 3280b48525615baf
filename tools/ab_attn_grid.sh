#!/bin/bash
# One-GPU A/B of the attention CTA order: LPT grid (heads, blocks) vs the earlier head-major grid
# (MALLEUS_ATTN_GRID_HEADMAJOR=1): attention parity tests, kernel microbenchmark, N = 1 step x 2 each.
set -u
P=${1:-r02r}
O=gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_gpu_kernels.py tests/test_gpu_gqa.py -k "attention or gqa" > $O/${P}_tests.log 2>&1; echo "tests rc $?"; tail -2 $O/${P}_tests.log
for v in lpt headmajor; do
  if [ $v = headmajor ]; then export MALLEUS_ATTN_GRID_HEADMAJOR=1; else unset MALLEUS_ATTN_GRID_HEADMAJOR; fi
  timeout 300 python tools/attn_bench.py > $O/${P}_attn_$v.log 2>&1; echo "attn $v rc $?"; cat $O/${P}_attn_$v.log | grep "nb="
done
for k in 1 2; do
for v in lpt headmajor; do
  if [ $v = headmajor ]; then export MALLEUS_ATTN_GRID_HEADMAJOR=1; else unset MALLEUS_ATTN_GRID_HEADMAJOR; fi
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/${P}_n1_${v}_$k.json 2> $O/${P}_n1_${v}_$k.err; echo "n1 $v $k rc $?"
  python -c "
import json; d=json.loads(open('$O/${P}_n1_${v}_$k.json').read().strip().splitlines()[-1]); print('n1 $v $k', round(d['value']), round(d['instrumentation']['tokens_s_same_steps_without_events']), round(d['ms_per_step'], 2), d['clocks']['sm_mhz'])"
done
done
