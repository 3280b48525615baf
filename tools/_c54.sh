mkdir -p gpurun_out
S=gpurun_out/c54_status
timeout 900 python -m pytest tests/test_gpu_step.py -x -q -k "P1 or P2 or P8 or peer or scatter or P3" > gpurun_out/c54_step.log 2>&1; echo step $? >> $S
MALLEUS_WATCHDOG=250 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29622 bench.py --gpus 2 --steps 10 --warmup 3 --no-straggler --uniform > gpurun_out/c54_t0_2.log 2>&1; echo t0_2 $? >> $S
MALLEUS_TP_NO_OVERLAP=1 MALLEUS_WATCHDOG=250 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29623 bench.py --gpus 2 --steps 10 --warmup 3 --no-straggler --uniform > gpurun_out/c54_t0_2_noov.log 2>&1; echo t0_2_noov $? >> $S
MALLEUS_WATCHDOG=250 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29624 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/c54_bench2.log 2>&1; echo bench2 $? >> $S
cat $S
