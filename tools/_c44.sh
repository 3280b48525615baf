mkdir -p gpurun_out
S=gpurun_out/c44_status
timeout 300 python -m pytest tests/test_gpu_tp_reduce.py -x -q > gpurun_out/c44_tpr.log 2>&1; echo tpr $? >> $S
timeout 1200 python -m pytest tests/test_gpu_step.py tests/test_gpu_kernels.py -x -q -k "scatter or peer or P1 or P2 or P4 or P9 or P3 or rmsnorm" > gpurun_out/c44_step.log 2>&1; echo step $? >> $S
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29671 tools/tp_step_trace.py > gpurun_out/c44_tptrace.log 2>&1; echo trace $? >> $S
for n in 2 4; do
MALLEUS_WATCHDOG=250 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2962$n bench.py --gpus $n --steps 10 --warmup 3 --no-straggler --uniform > gpurun_out/c44_t0_$n.log 2>&1; echo t0_$n $? >> $S
MALLEUS_WATCHDOG=250 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2963$n bench.py --gpus $n --steps 10 --warmup 3 > gpurun_out/c44_bench$n.log 2>&1; echo bench$n $? >> $S
done
cat $S
