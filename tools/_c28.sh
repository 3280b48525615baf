mkdir -p gpurun_out
S=gpurun_out/c28_status
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k attention > gpurun_out/c28_kern.log 2>&1; echo kern $? >> $S
for p in 0 2 3 4; do echo "POLY=$p" >> gpurun_out/c28_attn.log; MALLEUS_ATTN_POLY=$p timeout 120 python tools/attn_bench.py >> gpurun_out/c28_attn.log 2>&1; done; echo attn $? >> $S
timeout 120 python tools/attn_trace.py > gpurun_out/c28_trace.log 2>&1; echo trace $? >> $S
cat $S
