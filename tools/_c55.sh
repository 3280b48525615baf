mkdir -p gpurun_out
S=gpurun_out/c55_status
MALLEUS_WATCHDOG=250 timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/c55_bench1.log 2>&1; echo bench1 $? >> $S
MALLEUS_WATCHDOG=250 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29614 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/c55_bench4.log 2>&1; echo bench4 $? >> $S
timeout 240 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/c55_smoke.log 2>&1; echo smoke $? >> $S
timeout 840 python -m pytest tests -q -m gpu > gpurun_out/c55_tests.log 2>&1; echo tests $? >> $S
cat $S
