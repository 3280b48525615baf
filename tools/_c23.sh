set -x
mkdir -p gpurun_out
S=gpurun_out/c23_status
timeout 300 python -m pytest tests/test_gpu_tp_reduce.py -x -q > gpurun_out/c23_tpr.log 2>&1; echo tpr $? >> $S
timeout 200 python tools/tp_bench.py > gpurun_out/c23_tpbench.log 2>&1; echo tpbench $? >> $S
cat $S
