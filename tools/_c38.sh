mkdir -p gpurun_out
S=gpurun_out/c38_status
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_step.py -x -q -k "not P4 and not P5 and not P6 and not P7" > gpurun_out/c38_tests.log 2>&1; echo tests $? >> $S
MALLEUS_WATCHDOG=250 timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c38_bench1.log 2>&1; echo bench1 $? >> $S
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 5600 -c 2000 --csv --log-file gpurun_out/c38_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/c38_ncu.log 2>&1; echo launches $? >> $S
cat $S
