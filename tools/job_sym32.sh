# sym_pass32 with the whole coupling block prefetched: stage times + hgemv, then the parity suites
mkdir -p gpurun_out
for c in cfg2b1 cfg1; do
timeout 600 python tools/order_probe.py --config $c --combos 1:0:1:1,1:0:1:0,1:0:1:1 --reps 50 > gpurun_out/sym32_$c.txt 2>&1
done
timeout 900 python -m pytest tests/test_hgemv_gpu.py tests/test_core_gpu.py tests/test_dist_gpu.py tests/test_hara_gpu.py tests/test_inversion_gpu.py -x -q > gpurun_out/pytest_sym32.txt 2>&1; echo "exit $?" >> gpurun_out/pytest_sym32.txt
timeout 600 python bench.py --config cfg2b1 --steps 20 --warmup 3 > gpurun_out/bench_cfg2b1_sym32.json 2> /dev/null
tail -n 3 gpurun_out/sym32_*.txt gpurun_out/pytest_sym32.txt
