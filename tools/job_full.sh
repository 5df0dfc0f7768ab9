export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_full.txt 2>&1; echo "exit $?" >> gpurun_out/pytest_full.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_full.txt 2>&1; echo "exit $?" >> gpurun_out/smoke_full.txt
timeout 600 python bench.py --config cfg3 --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/bench_cfg3_reg.json 2> gpurun_out/bench_cfg3_reg.err
ncu --kernel-name-base demangled --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"carry|cn_step|hess_finish|nu_rowmajor" --csv --log-file gpurun_out/diff_launches_reg.csv python tools/diff1d_probe.py --b 16 --reps 1 --check 0 > gpurun_out/diff_launch_reg.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:cn_step_kernel --launch-skip 100 -c 1 -o gpurun_out/diff_reg1 python tools/diff1d_probe.py --b 16 --reps 1 --check 0 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:cn_step_kernel --launch-skip 180 -c 1 -o gpurun_out/diff_reg2 python tools/diff1d_probe.py --b 16 --reps 1 --check 0 > /dev/null 2>&1
