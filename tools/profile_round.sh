#!/bin/bash
# One-GPU evidence pass (run on the GPU box from the repo root): bench line, launch list, per-shape
# GEMM metrics, attention timing + ncu captures, compute-sanitizer checks.  Outputs in gpurun_out/$1_*.
set -u
P=${1:-r02j}
O=gpurun_out
python bench.py --steps 20 --warmup 5 > $O/${P}_bench.json 2> $O/${P}_bench.err; echo "bench rc $?"; tail -c 600 $O/${P}_bench.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/${P}_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/${P}_ncu_launches.log 2>&1; echo "launch list rc $?"
rm -f $O/${P}_gemm_log.txt
MALLEUS_GEMM_LOG=$O/${P}_gemm_log.txt ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:gemm_tcgen05 --launch-skip 2448 --launch-count 816 --csv --log-file $O/${P}_gemm_shapes.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/${P}_ncu_gemm.log 2>&1; echo "gemm shapes rc $?"
python tools/attn_bench.py > $O/${P}_attn_bench.log 2>&1; echo "attn bench rc $?"; cat $O/${P}_attn_bench.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_ --launch-skip 4 --launch-count 4 \
    -o $O/${P}_ncu_attn python tools/attn_one.py > $O/${P}_ncu_attn.log 2>&1; echo "attn ncu rc $?"
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard python -m pytest tests/test_gpu_tp_reduce.py -x -q -m gpu -k "one_device" > $O/${P}_racecheck_tp.log 2>&1; echo "racecheck tp rc $?"; tail -5 $O/${P}_racecheck_tp.log
timeout 900 compute-sanitizer --tool synccheck python -m pytest tests/test_gpu_tp_reduce.py -x -q -m gpu -k "one_device" > $O/${P}_synccheck_tp.log 2>&1; echo "synccheck tp rc $?"; tail -5 $O/${P}_synccheck_tp.log
timeout 1200 compute-sanitizer --tool memcheck python -c "import __graft_entry__ as g; g.smoke()" > $O/${P}_memcheck_smoke.log 2>&1; echo "memcheck smoke rc $?"; tail -5 $O/${P}_memcheck_smoke.log
timeout 1200 compute-sanitizer --tool racecheck python -c "import __graft_entry__ as g; g.smoke()" > $O/${P}_racecheck_smoke.log 2>&1; echo "racecheck smoke rc $?"; tail -5 $O/${P}_racecheck_smoke.log
