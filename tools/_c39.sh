mkdir -p gpurun_out
S=gpurun_out/c39_status
nvidia-smi -L > gpurun_out/c39_gpus.log
timeout 900 python -m pytest tests/test_gpu_step.py -x -q -k "P7" > gpurun_out/c39_p7.log 2>&1; echo p7 $? >> $S
MALLEUS_WATCHDOG=250 timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29618 bench.py --gpus 8 --steps 10 --warmup 3 > gpurun_out/c39_bench8.log 2>&1; echo bench8 $? >> $S
MALLEUS_WATCHDOG=250 timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29628 bench.py --gpus 8 --steps 10 --warmup 3 --no-straggler --uniform > gpurun_out/c39_t0_8.log 2>&1; echo t0_8 $? >> $S
MALLEUS_WATCHDOG=250 timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29638 bench.py --gpus 8 --steps 10 --warmup 3 --uniform --no-replan > gpurun_out/c39_tu_8.log 2>&1; echo tu_8 $? >> $S
cat $S
