mkdir -p gpurun_out
S=gpurun_out/c51_status
timeout 900 python -m pytest tests/test_gpu_step.py -x -q -k "clipping or p0 or P4 or bitwise or P9" > gpurun_out/c51_step.log 2>&1; echo step $? >> $S
MALLEUS_WATCHDOG=250 timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c51_bench1.log 2>&1; echo bench1 $? >> $S
cat $S
