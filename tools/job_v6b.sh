export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
nproc > gpurun_out/host_v6b.txt; lscpu | grep -i "model name\|numa\|socket" >> gpurun_out/host_v6b.txt; nvidia-smi topo -m >> gpurun_out/host_v6b.txt 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_cfg2_v6b.json 2> gpurun_out/bench_cfg2_v6b.err
timeout 600 python bench.py --config cfg3k --steps 7 --warmup 2 --no-cpu-baseline > gpurun_out/bench_cfg3k_v6b.json 2> gpurun_out/bench_cfg3k_v6b.err
timeout 300 python tools/diff1d_probe.py --b 16 64 --check 0 > gpurun_out/diff_probe_v6b.txt 2>&1
bash tools/diff_prof.sh
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"carry|cn_step|hess_finish|nu_rowmajor" --csv --log-file gpurun_out/diff_launches_v6b.csv python tools/diff1d_probe.py --b 16 --reps 1 --check 0 > gpurun_out/diff_launch_v6b.log 2>&1
