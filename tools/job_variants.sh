mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
cp paper_2003_10173_b200/lib/libh2b200.so /tmp/default.so
for v in acc4 acc2; do
  cp tools/variants/$v.so paper_2003_10173_b200/lib/libh2b200.so
  echo "== $v" >> gpurun_out/variants.txt
  timeout 300 python tools/diff1d_probe.py --b 16 64 --check 0 >> gpurun_out/variants.txt 2>&1
  ncu --kernel-name-base demangled --metrics gpu__time_duration.sum --clock-control none -k regex:"cn_step_kernel<2>" -c 20 --csv --log-file gpurun_out/var_$v.csv python tools/diff1d_probe.py --b 16 --reps 1 --check 0 > /dev/null 2>&1
done
cp /tmp/default.so paper_2003_10173_b200/lib/libh2b200.so
