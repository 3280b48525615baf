mkdir -p gpurun_out
S=gpurun_out/c30_status
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k attention > gpurun_out/c30_kern.log 2>&1; echo kern $? >> $S
timeout 120 python tools/attn_bench.py > gpurun_out/c30_attn.log 2>&1; echo attn $? >> $S
timeout 600 python -m pytest tests/test_gpu_step.py -x -q -k "p0" > gpurun_out/c30_step.log 2>&1; echo step $? >> $S
cat $S
