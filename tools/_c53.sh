mkdir -p gpurun_out
S=gpurun_out/c53_status
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k attention > gpurun_out/c53_kern.log 2>&1; echo kern $? >> $S
for p in 0 1 2 3; do MALLEUS_ATTN_POLY=$p timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attn_fwd" --csv python tools/attn_one.py > gpurun_out/c53_ncu_$p.csv 2>&1; echo ncu$p $? >> $S; done
cat $S
