#!/bin/bash
# Final one-GPU pass: smoke, bench line (with the oracle baseline), ncu launch list of one step.
set -u
P=${1:-r02final}
O=gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > $O/${P}_smoke.log 2>&1; echo "smoke rc $?"; tail -2 $O/${P}_smoke.log
python bench.py --steps 20 --warmup 5 > $O/${P}_bench_n1.json 2> $O/${P}_bench_n1.err; echo "bench rc $?"; tail -c 900 $O/${P}_bench_n1.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/${P}_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/${P}_ncu_launches.log 2>&1; echo "launch list rc $?"
python bench.py --impl reference --steps 3 --warmup 1 > $O/${P}_reference.json 2>&1; echo "reference rc $?"; tail -c 400 $O/${P}_reference.json
