#!/bin/bash
# Two-GPU confirmation pass of the last build: step parity on <= 2 GPUs (incl. pair mode on a TP-2
# stage), kernel tests, the N = 2 straggler line, smoke.
set -u
P=${1:-r02w}
O=gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > $O/${P}_smoke.log 2>&1; echo "smoke rc $?"; tail -1 $O/${P}_smoke.log
timeout 1200 python -m pytest -q -m gpu tests/test_gpu_step.py tests/test_gpu_kernels.py tests/test_gpu_layer_api.py > $O/${P}_tests.log 2>&1; echo "tests rc $?"; tail -2 $O/${P}_tests.log
CUDA_VISIBLE_DEVICES=0,1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29571 bench.py --gpus 2 --steps 10 --warmup 3 > $O/${P}_bench_n2.json 2> $O/${P}_bench_n2.err; echo "n2 rc $?"
python -c "
import json; d=json.loads(open('$O/${P}_bench_n2.json').read().strip().splitlines()[-1]); print('n2', round(d['value']), round(d['instrumentation']['tokens_s_same_steps_without_events']), {k: round(v) for k, v in d['baselines'].items() if k.endswith('tokens_s')}, d['straggling_measured'], [(c['plan'][0]['stages'][0]['heads'], round(c['tokens_s'])) for c in d['replan']['candidates']], d['replan']['replanned_plan'], d['clocks'], d['roofline'])"
