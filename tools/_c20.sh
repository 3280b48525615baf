set -x
mkdir -p gpurun_out
S=gpurun_out/c20_status
timeout 400 python -m pytest tests/test_gpu_kernels.py -x -q -k attention > gpurun_out/c20_kern.log 2>&1; echo kern $? >> $S
timeout 120 python tools/attn_bench.py > gpurun_out/c20_attn.log 2>&1; echo attn $? >> $S
timeout 900 python -m pytest tests/test_gpu_step.py -x -q -k "p0 or d128 or peer or P1 or P2 or P3 or P8" > gpurun_out/c20_step.log 2>&1; echo step $? >> $S
MALLEUS_WATCHDOG=250 timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/c20_bench1.log 2>&1; echo bench1 $? >> $S
MALLEUS_WATCHDOG=250 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/c20_bench2.log 2>&1; echo bench2 $? >> $S
MALLEUS_WATCHDOG=250 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 2 --steps 10 --warmup 3 --no-straggler --no-replan > gpurun_out/c20_t0_2.log 2>&1; echo t0_2 $? >> $S
cat $S
