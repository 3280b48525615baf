#!/bin/bash
# Two-GPU A/B pass: RMSNorm backward row-group kernel (parity tests + microbench + N = 1 step with and
# without it) and pair mode at N = 2 under the straggler (MALLEUS_WGRAD_PAIR_OFF=1 vs default).
set -u
P=${1:-r02x}
O=gpurun_out
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest -q -m gpu tests/test_gpu_kernels.py tests/test_gpu_c2_full.py > $O/${P}_tests.log 2>&1; echo "tests rc $?"; tail -2 $O/${P}_tests.log
CUDA_VISIBLE_DEVICES=0 timeout 600 python tools/norm_bwd_bench.py > $O/${P}_norm_bwd_bench.log 2>&1; echo "norm bench rc $?"; cat $O/${P}_norm_bwd_bench.log | head -4
for v in rows block; do
  if [ $v = block ]; then export MALLEUS_NORM_BWD_BLOCK=1; else unset MALLEUS_NORM_BWD_BLOCK; fi
  CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/${P}_n1_$v.json 2> $O/${P}_n1_$v.err; echo "n1 $v rc $?"
  python -c "
import json; d=json.loads(open('$O/${P}_n1_$v.json').read().strip().splitlines()[-1]); print('n1 $v', round(d['value']), round(d['instrumentation']['tokens_s_same_steps_without_events']), d['clocks'], d['roofline']['frac'], d['roofline'].get('frac_at_run_clock'))"
done
unset MALLEUS_NORM_BWD_BLOCK
for v in nopair pair; do
  if [ $v = nopair ]; then export MALLEUS_WGRAD_PAIR_OFF=1; else unset MALLEUS_WGRAD_PAIR_OFF; fi
  CUDA_VISIBLE_DEVICES=0,1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29591 bench.py --gpus 2 --steps 10 --warmup 3 > $O/${P}_n2_$v.json 2> $O/${P}_n2_$v.err; echo "n2 $v rc $?"
  python -c "
import json; d=json.loads(open('$O/${P}_n2_$v.json').read().strip().splitlines()[-1]); print('n2 $v', round(d['value']), round(d['instrumentation']['tokens_s_same_steps_without_events']), {k: round(v) for k, v in d['baselines'].items() if k.endswith('tokens_s')}, d['straggling_measured']['pass_probe'], d['straggling_measured']['pass_nominal'], d['straggling_measured']['x_probe'], [(c['plan'][0]['stages'][0]['heads'], round(c['tokens_s'])) for c in d['replan']['candidates']], round(d['replan']['tokens_s_before']), d['replan']['compute_ms_per_rank_before'], d['clocks'])"
done
