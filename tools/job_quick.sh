mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_hgemv_gpu.py tests/test_core_gpu.py tests/test_dist_gpu.py tests/test_hara_gpu.py -x -q > gpurun_out/pytest_quick.txt 2>&1; echo "exit $?" >> gpurun_out/pytest_quick.txt
for c in cfg2b1 cfg1 cfg2; do
timeout 600 python tools/order_probe.py --config $c --combos 1:0:1,1:0:1 --reps 20 > gpurun_out/quick_$c.txt 2>&1
done
