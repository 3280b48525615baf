#!/bin/bash
# Four-GPU pass of the last build: the N = 4 straggler line, the dynamic trace, the >2-GPU step parity plans.
set -u
P=${1:-r02v}
O=gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 --master-port=29572 bench.py --gpus 4 --steps 10 --warmup 3 > $O/${P}_bench_n4.json 2> $O/${P}_bench_n4.err; echo "n4 rc $?"
python -c "
import json; d=json.loads(open('$O/${P}_bench_n4.json').read().strip().splitlines()[-1]); print('n4', round(d['value']), round(d['instrumentation']['tokens_s_same_steps_without_events']), {k: round(v) for k, v in d['baselines'].items() if k.endswith('tokens_s')}, d['straggling_measured'], [(c['plan'], round(c['tokens_s'])) for c in d['replan']['candidates']], d['replan']['replanned_plan'], d['clocks'])"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 --master-port=29574 tools/trace_run.py --out $O/${P}_trace.json > $O/${P}_trace.log 2>&1; echo "trace rc $?"; grep '"situation"' $O/${P}_trace.log | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['situation'], d['x_probed'], d['standby'], d['plan'], d['ms_stale_plan'], d['ms_replanned'], d['refined_from_measured_compute'], d['R_opt_over_R_actual'])"
timeout 900 python -m pytest -q -m gpu tests/test_gpu_step.py -k "P4 or P5 or P6 or P9 or P11" > $O/${P}_tests.log 2>&1; echo "tests rc $?"; tail -2 $O/${P}_tests.log
