mkdir -p gpurun_out
cp paper_2003_10173_b200/lib/libh2b200.so /tmp/default.so
for v in seg32only both seg32only both; do
  cp tools/variants/$v.so paper_2003_10173_b200/lib/libh2b200.so
  echo "== $v" >> gpurun_out/variants.txt
  for c in cfg2 cfg4; do timeout 300 python tools/order_probe.py --config $c --combos 1:0:1 --reps 10 >> gpurun_out/variants.txt 2>&1; done
done
cp /tmp/default.so paper_2003_10173_b200/lib/libh2b200.so
timeout 600 python -m pytest tests/test_hgemv_gpu.py tests/test_dist_gpu.py tests/test_core_gpu.py -x -q 2>&1 | tail -1 >> gpurun_out/variants.txt
