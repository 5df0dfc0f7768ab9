mkdir -p gpurun_out
timeout 600 python tools/order_probe.py --combos 0:0,1:0,1:1,0:1 > gpurun_out/order_probe.txt 2>&1
timeout 900 ncu --kernel-name-base demangled --kernel-name regex:"seg_gemm_kernel" --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/order_ncu.csv python tools/order_probe.py --combos 0:0,1:0,1:1 --no-stages --reps 1 > gpurun_out/order_ncu.log 2>&1
echo done >> gpurun_out/order_probe.txt
