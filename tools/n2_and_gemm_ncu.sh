#!/bin/bash
# Two-GPU pass: the N = 2 straggler line (measured re-split candidates), then on GPU 0 one ncu
# metrics capture of every GEMM launch of one N = 1 step (pair build: 680 per step) joined with the
# MALLEUS_GEMM_LOG shape log -> per-shape table and the bench's roofline.traffic file.
set -u
P=${1:-r02y}
O=gpurun_out
CUDA_VISIBLE_DEVICES=0,1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29581 bench.py --gpus 2 --steps 10 --warmup 3 > $O/${P}_bench_n2.json 2> $O/${P}_bench_n2.err; echo "n2 rc $?"
python -c "
import json; d=json.loads(open('$O/${P}_bench_n2.json').read().strip().splitlines()[-1]); print('n2', round(d['value']), {k: round(v) for k, v in d['baselines'].items() if k.endswith('tokens_s')}, d['straggling_measured'], d['replan'], d['clocks'])"
rm -f $O/${P}_gemm_log.txt
CUDA_VISIBLE_DEVICES=0 MALLEUS_GEMM_LOG=$O/${P}_gemm_log.txt timeout 1200 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:gemm_tcgen05 --launch-skip 2040 --launch-count 680 --csv --log-file $O/${P}_gemm_m.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/${P}_gemm_ncu.log 2>&1; echo "gemm ncu rc $?"
python tools/gemm_shapes_report.py $O/${P}_gemm_m.csv $O/${P}_gemm_log.txt 2040 > $O/${P}_gemm_shapes.md; echo "report rc $?"
python tools/gemm_traffic_from_shapes.py $O/${P}_gemm_m.csv $O/${P}_gemm_log.txt 2040 > $O/${P}_gemm_traffic.json; echo "traffic rc $?"; cat $O/${P}_gemm_traffic.json
