mkdir -p gpurun_out
S=gpurun_out/c52_status
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k attention > gpurun_out/c52_kern.log 2>&1; echo kern $? >> $S
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attn_" --csv python tools/attn_one.py > gpurun_out/c52_ncu.csv 2>&1; echo ncu $? >> $S
timeout 120 python tools/attn_trace.py > gpurun_out/c52_trace.log 2>&1; echo trace $? >> $S
timeout 600 python -m pytest tests/test_gpu_step.py -x -q -k "p0" > gpurun_out/c52_step.log 2>&1; echo step $? >> $S
cat $S
