mkdir -p gpurun_out
S=gpurun_out/c37_status
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/c37_plain.log 2>&1; echo plain $? >> $S
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 5600 -c 2000 --csv --log-file gpurun_out/c37_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/c37_ncu.log 2>&1; echo launches $? >> $S
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gemm -s 2448 -c 816 --csv --log-file gpurun_out/c37_gemm_dram.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/c37_ncu2.log 2>&1; echo dram $? >> $S
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"attn_|tp_reduce|rmsnorm_bwd" -s 20 -c 4 -o gpurun_out/c37_attn_full -f python tools/attn_one.py > gpurun_out/c37_ncu3.log 2>&1; echo full $? >> $S
cat $S
