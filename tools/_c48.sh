mkdir -p gpurun_out
S=gpurun_out/c48_status
MALLEUS_WATCHDOG=250 timeout 400 python bench.py --steps 10 --warmup 3 > gpurun_out/c48_bench1.log 2>&1; echo bench1 $? >> $S
for n in 2 4; do
MALLEUS_WATCHDOG=250 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2961$n bench.py --gpus $n --steps 10 --warmup 3 > gpurun_out/c48_bench$n.log 2>&1; echo bench$n $? >> $S
MALLEUS_WATCHDOG=250 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2962$n bench.py --gpus $n --steps 10 --warmup 3 --no-straggler --uniform > gpurun_out/c48_t0_$n.log 2>&1; echo t0_$n $? >> $S
MALLEUS_WATCHDOG=250 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2963$n bench.py --gpus $n --steps 10 --warmup 3 --uniform --no-replan > gpurun_out/c48_tu_$n.log 2>&1; echo tu_$n $? >> $S
done
MALLEUS_WATCHDOG=250 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29644 bench.py --gpus 4 --steps 10 --warmup 3 --tp4-stage > gpurun_out/c48_tp4.log 2>&1; echo tp4 $? >> $S
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/c48_smoke.log 2>&1; echo smoke $? >> $S
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/c48_tests.log 2>&1; echo tests $? >> $S
cat $S
