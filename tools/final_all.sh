#!/bin/bash
# Final pass on a 4-GPU box: the N = 2 / N = 4 straggler lines and the trace, the N = 1 line (GPU 0),
# smoke, launch list, reference arm, and the full GPU test suite.
set -u
bash tools/straggler_n4.sh r02z
CUDA_VISIBLE_DEVICES=0 bash tools/final_n1.sh r02z
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/r02z_tests.log 2>&1; echo "tests rc $?"; tail -3 gpurun_out/r02z_tests.log
