#!/bin/bash
# Final one-GPU evidence of the last build: smoke, the default bench line (with the oracle baseline),
# the whole -m gpu suite, the reference arm, and an ncu launch list of one step.
set -u
P=${1:-r02s}
O=gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > $O/${P}_smoke.log 2>&1; echo "smoke rc $?"; tail -1 $O/${P}_smoke.log
python bench.py > $O/${P}_bench_n1.json 2> $O/${P}_bench_n1.err; echo "bench rc $?"; tail -c 1500 $O/${P}_bench_n1.json
timeout 1500 python -m pytest -q -m gpu tests > $O/${P}_tests.log 2>&1; echo "tests rc $?"; tail -2 $O/${P}_tests.log
python bench.py --impl reference --steps 3 --warmup 1 > $O/${P}_reference.json 2>&1; echo "reference rc $?"; tail -c 300 $O/${P}_reference.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/${P}_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/${P}_ncu_launches.log 2>&1; echo "launch list rc $?"
