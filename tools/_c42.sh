mkdir -p gpurun_out
S=gpurun_out/c42_status
for i in 1 2; do
MALLEUS_WATCHDOG=250 timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c42_a$i.log 2>&1; echo a$i $? >> $S
MALLEUS_BENCH_NO_GEMM_EVENTS=1 MALLEUS_WATCHDOG=250 timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c42_b$i.log 2>&1; echo b$i $? >> $S
done
cat $S
