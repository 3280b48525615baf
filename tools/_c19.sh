set -x
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_kernels.py -x -q -k attention > gpurun_out/c19_kern.log 2>&1; echo kern $? >> gpurun_out/c19_status
timeout 120 python tools/attn_bench.py > gpurun_out/c19_attn.log 2>&1; echo attn $? >> gpurun_out/c19_status
timeout 400 python -m pytest tests/test_gpu_step.py -x -q -k "p0 or d128" > gpurun_out/c19_step.log 2>&1; echo step $? >> gpurun_out/c19_status
MALLEUS_WATCHDOG=250 timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/c19_bench1.log 2>&1; echo bench $? >> gpurun_out/c19_status
tail -3 gpurun_out/c19_*.log
