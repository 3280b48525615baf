#!/bin/bash
# Straggler evidence pass on 4 GPUs: N = 2 and N = 4 bench lines and the dynamic trace.
set -u
P=${1:-r02m}
O=gpurun_out
CUDA_VISIBLE_DEVICES=0,1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29571 bench.py --gpus 2 --steps 10 --warmup 3 > $O/${P}_bench_n2.json 2> $O/${P}_bench_n2.err; echo "n2 rc $?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 --master-port=29572 bench.py --gpus 4 --steps 10 --warmup 3 > $O/${P}_bench_n4.json 2> $O/${P}_bench_n4.err; echo "n4 rc $?"
for f in n2 n4; do python -c "
import json; d=json.loads(open('$O/${P}_bench_$f.json').read().strip().splitlines()[-1]); print('$f', round(d['value']), d['baselines'] and {k: round(v) for k, v in d['baselines'].items() if k.endswith('tokens_s')}, d['straggling_measured'], d['replan'] and d['replan']['replanned_plan'], d['clocks'])"; done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 --master-port=29574 tools/trace_run.py --out $O/${P}_trace.json > $O/${P}_trace.log 2>&1; echo "trace rc $?"; grep '"situation"' $O/${P}_trace.log | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['situation'], d['x_probed'], d['standby'], d['ms_stale_plan'], d['ms_replanned'], d['R_opt_over_R_actual'])"
