mkdir -p gpurun_out
S=gpurun_out/c36_status
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/c36_tests.log 2>&1; echo tests $? >> $S
MALLEUS_WATCHDOG=250 timeout 400 python bench.py --steps 10 --warmup 3 > gpurun_out/c36_bench1.log 2>&1; echo bench1 $? >> $S
for n in 2 4; do
MALLEUS_WATCHDOG=250 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2961$n bench.py --gpus $n --steps 10 --warmup 3 > gpurun_out/c36_bench$n.log 2>&1; echo bench$n $? >> $S
MALLEUS_WATCHDOG=250 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2962$n bench.py --gpus $n --steps 10 --warmup 3 --no-straggler --uniform --no-cpu-baseline > gpurun_out/c36_t0_$n.log 2>&1; echo t0_$n $? >> $S
MALLEUS_WATCHDOG=250 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2963$n bench.py --gpus $n --steps 10 --warmup 3 --uniform --no-replan --no-cpu-baseline > gpurun_out/c36_tu_$n.log 2>&1; echo tu_$n $? >> $S
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29650 tools/bench_migrate.py > gpurun_out/c36_mig.log 2>&1; echo mig $? >> $S
cat $S
