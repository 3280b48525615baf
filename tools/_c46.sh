mkdir -p gpurun_out
S=gpurun_out/c46_status
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k attention > gpurun_out/c46_kern.log 2>&1; echo kern $? >> $S
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attn_" --csv python tools/attn_one.py > gpurun_out/c46_ncu.csv 2>&1; echo ncu $? >> $S
timeout 600 python -m pytest tests/test_gpu_step.py -x -q -k "p0" > gpurun_out/c46_step.log 2>&1; echo step $? >> $S
MALLEUS_WATCHDOG=250 timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c46_bench1.log 2>&1; echo bench1 $? >> $S
cat $S
