#!/bin/bash
# One-GPU A/B: pair-flush weight-gradient GEMMs on a side stream (default) vs on the main stream
# (MALLEUS_WGRAD_SIDE_OFF=1), after the step parity tests that exercise pair mode at TP 1.
set -u
P=${1:-r02t}
O=gpurun_out
timeout 1200 python -m pytest -q -m gpu tests/test_gpu_step.py tests/test_gpu_c2_full.py tests/test_gpu_gqa.py tests/test_gpu_layer_api.py > $O/${P}_tests.log 2>&1; echo "tests rc $?"; tail -2 $O/${P}_tests.log
for k in 1 2; do
for v in side main; do
  if [ $v = main ]; then export MALLEUS_WGRAD_SIDE_OFF=1; else unset MALLEUS_WGRAD_SIDE_OFF; fi
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/${P}_n1_${v}_$k.json 2> $O/${P}_n1_${v}_$k.err; echo "n1 $v $k rc $?"
  python -c "
import json; d=json.loads(open('$O/${P}_n1_${v}_$k.json').read().strip().splitlines()[-1]); r=d['roofline']; print('n1 $v $k', round(d['value']), round(d['instrumentation']['tokens_s_same_steps_without_events']), round(d['ms_per_step'], 2), d['clocks']['sm_mhz'], round(r['achieved']), round(r['frac'], 3), round(r['gemm_share_of_step'], 3), d['e2e']['value'])"
done
done
