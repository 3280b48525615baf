set -x
mkdir -p gpurun_out
S=gpurun_out/c26_status
timeout 300 python -m pytest tests/test_gpu_tp_reduce.py -x -q > gpurun_out/c26_tpr.log 2>&1; echo tpr $? >> $S
MALLEUS_TP_TRACE=1 timeout 200 python tools/tp_bench.py > gpurun_out/c26_tpbench.log 2>&1; echo tpbench $? >> $S
TP_BF16=1 timeout 200 python tools/tp_bench.py > gpurun_out/c26_tpbench_bf16.log 2>&1; echo tpbench16 $? >> $S
timeout 600 python -m pytest tests/test_gpu_step.py -x -q -k "peer or P2 or P1" > gpurun_out/c26_step.log 2>&1; echo step $? >> $S
MALLEUS_TP_PARTIAL=bf16 timeout 600 python -m pytest tests/test_gpu_step.py -x -q -k "P2 or P1 or P4 or P3 or P8" > gpurun_out/c26_step16.log 2>&1; echo step16 $? >> $S
for n in 2 4; do
MALLEUS_WATCHDOG=250 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2962$n bench.py --gpus $n --steps 10 --warmup 3 --no-straggler --uniform --no-cpu-baseline > gpurun_out/c26_t0_$n.log 2>&1; echo t0_$n $? >> $S
MALLEUS_TP_PARTIAL=bf16 MALLEUS_WATCHDOG=250 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2963$n bench.py --gpus $n --steps 10 --warmup 3 --no-straggler --uniform --no-cpu-baseline > gpurun_out/c26_t0_${n}_bf16.log 2>&1; echo t0_${n}_bf16 $? >> $S
done
cat $S
