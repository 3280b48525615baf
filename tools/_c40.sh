mkdir -p gpurun_out
S=gpurun_out/c40_status
timeout 900 python -m pytest tests/test_gpu_step.py -x -q -k "P9" > gpurun_out/c40_p9.log 2>&1; echo p9 $? >> $S
MALLEUS_WATCHDOG=250 timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29614 bench.py --gpus 4 --steps 10 --warmup 3 --tp4-stage > gpurun_out/c40_tp4.log 2>&1; echo tp4 $? >> $S
MALLEUS_WATCHDOG=250 timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29624 bench.py --gpus 4 --steps 10 --warmup 3 --tp4-stage --no-straggler --uniform > gpurun_out/c40_tp4_t0.log 2>&1; echo tp4_t0 $? >> $S
MALLEUS_WATCHDOG=250 timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29634 bench.py --gpus 4 --steps 10 --warmup 3 --tp4-stage --uniform --no-replan > gpurun_out/c40_tp4_tu.log 2>&1; echo tp4_tu $? >> $S
cat $S
