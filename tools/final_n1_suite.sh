#!/bin/bash
# One-GPU pass: attention backward dQ || dK/dV concurrency A/B on the N = 1 step (two runs each,
# alternating), then the whole -m gpu suite as the driver's 1-GPU box runs it, and smoke.
set -u
P=${1:-r02u}
O=gpurun_out
for k in 1 2; do
for v in conc serial; do
  if [ $v = serial ]; then export MALLEUS_ATTN_BWD_SERIAL=1; else unset MALLEUS_ATTN_BWD_SERIAL; fi
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/${P}_n1_${v}_$k.json 2> $O/${P}_n1_${v}_$k.err; echo "n1 $v $k rc $?"
  python -c "
import json; d=json.loads(open('$O/${P}_n1_${v}_$k.json').read().strip().splitlines()[-1]); print('n1 $v $k', round(d['value']), round(d['instrumentation']['tokens_s_same_steps_without_events']), round(d['ms_per_step'], 2), d['clocks']['sm_mhz'], d['breakdown_ms_rank0'])"
done
done
unset MALLEUS_ATTN_BWD_SERIAL
python -c "import __graft_entry__ as g; g.smoke()" > $O/${P}_smoke.log 2>&1; echo "smoke rc $?"; tail -1 $O/${P}_smoke.log
timeout 1800 python -m pytest -q -m gpu tests > $O/${P}_tests.log 2>&1; echo "tests rc $?"; tail -3 $O/${P}_tests.log
