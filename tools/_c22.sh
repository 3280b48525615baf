set -x
mkdir -p gpurun_out
S=gpurun_out/c22_status
timeout 200 python tools/tp_bench.py > gpurun_out/c22_tpbench.log 2>&1; echo tpbench $? >> $S
for n in 2 4; do
MALLEUS_WATCHDOG=250 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2962$n bench.py --gpus $n --steps 10 --warmup 3 --no-straggler --uniform --no-cpu-baseline > gpurun_out/c22_t0_$n.log 2>&1; echo t0_$n $? >> $S
MALLEUS_NO_P2P=1 MALLEUS_WATCHDOG=250 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2963$n bench.py --gpus $n --steps 10 --warmup 3 --no-straggler --uniform --no-cpu-baseline > gpurun_out/c22_t0_${n}_nop2p.log 2>&1; echo t0_${n}_nop2p $? >> $S
MALLEUS_WATCHDOG=250 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2964$n bench.py --gpus $n --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c22_s_$n.log 2>&1; echo s_$n $? >> $S
done
cat $S
