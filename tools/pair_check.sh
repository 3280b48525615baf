#!/bin/bash
# Pair-mode weight gradients: step parity over the plan matrix (1-4 GPUs), full-size C2 parity,
# and the N = 1 bench line with and without pairing.
set -u
P=${1:-r02t}
O=gpurun_out
timeout 1800 python -m pytest tests/test_gpu_step.py tests/test_gpu_c2_full.py tests/test_gpu_layer_api.py tests/test_gpu_gqa.py -q -m gpu -x > $O/${P}_tests.log 2>&1; echo "tests rc $?"; tail -3 $O/${P}_tests.log
CUDA_VISIBLE_DEVICES=0 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/${P}_bench_pair.json 2>&1; echo "pair rc $?"
CUDA_VISIBLE_DEVICES=0 MALLEUS_WGRAD_PAIR_OFF=1 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/${P}_bench_nopair.json 2>&1; echo "nopair rc $?"
for f in pair nopair; do python -c "
import json; d=json.loads(open('$O/${P}_bench_$f.json').read().strip().splitlines()[-1]); print('$f', round(d['value']), round(d['instrumentation']['tokens_s_same_steps_without_events']), d['ms_per_step'], d['clocks']['sm_mhz'], d['gpu_launches'])"; done
