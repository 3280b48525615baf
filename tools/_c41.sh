mkdir -p gpurun_out
S=gpurun_out/c41_status
timeout 600 python -m pytest tests/test_gpu_gemm.py -x -q > gpurun_out/c41_gemm.log 2>&1; echo gemm $? >> $S
timeout 1200 python -m pytest tests/test_gpu_step.py -x -q -k "scatter or peer or P2 or P4 or P9 or p0" > gpurun_out/c41_step.log 2>&1; echo step $? >> $S
for n in 2 4; do
MALLEUS_WATCHDOG=250 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2962$n bench.py --gpus $n --steps 10 --warmup 3 --no-straggler --uniform --no-cpu-baseline > gpurun_out/c41_t0_$n.log 2>&1; echo t0_$n $? >> $S
done
MALLEUS_WATCHDOG=250 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29644 bench.py --gpus 4 --steps 10 --warmup 3 --tp4-stage --no-straggler --uniform > gpurun_out/c41_tp4_t0.log 2>&1; echo tp4_t0 $? >> $S
MALLEUS_WATCHDOG=250 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29652 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/c41_bench2.log 2>&1; echo bench2 $? >> $S
cat $S
