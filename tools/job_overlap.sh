# few-vector hgemv: dense near-field pass concurrent with the sweep chain (h2b_tune 8) vs serial
mkdir -p gpurun_out
for c in cfg2b1 cfg1; do
timeout 600 python tools/order_probe.py --config $c --combos 1:0:1:0,1:0:1:1,1:0:1:0,1:0:1:1 --reps 50 > gpurun_out/overlap_$c.txt 2>&1
done
timeout 900 python -m pytest tests/test_hgemv_gpu.py tests/test_core_gpu.py tests/test_dist_gpu.py -x -q > gpurun_out/pytest_overlap.txt 2>&1; echo "exit $?" >> gpurun_out/pytest_overlap.txt
timeout 600 python bench.py --config cfg2b1 --steps 20 --warmup 3 > gpurun_out/bench_cfg2b1_overlap.json 2> gpurun_out/bench_cfg2b1_overlap.err
tail -n 3 gpurun_out/overlap_*.txt gpurun_out/pytest_overlap.txt
