set -x
mkdir -p gpurun_out
S=gpurun_out/c21_status
timeout 300 python -m pytest tests/test_gpu_tp_reduce.py -x -q > gpurun_out/c21_tpr.log 2>&1; echo tpr $? >> $S
timeout 200 python tools/tp_bench.py > gpurun_out/c21_tpbench.log 2>&1; echo tpbench $? >> $S
MALLEUS_WATCHDOG=250 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 2 --steps 10 --warmup 3 --no-straggler --no-replan > gpurun_out/c21_t0_2.log 2>&1; echo t0_2 $? >> $S
MALLEUS_NO_P2P=1 MALLEUS_WATCHDOG=250 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29613 bench.py --gpus 2 --steps 10 --warmup 3 --no-straggler --no-replan > gpurun_out/c21_t0_2_nop2p.log 2>&1; echo t0_2_nop2p $? >> $S
cat $S
