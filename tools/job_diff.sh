export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_diffusion_gpu.py tests/test_hara_gpu.py -x -q > gpurun_out/pytest_diff.txt 2>&1; echo "exit $?" >> gpurun_out/pytest_diff.txt
timeout 300 python tools/diff1d_probe.py --b 16 64 --check 2 --tune -1:0 -2:0 -1:0 > gpurun_out/diff_probe.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"carry|cn_step" -c 400 --csv --log-file gpurun_out/diff_launches.csv python tools/diff1d_probe.py --b 16 --reps 1 --check 0 > gpurun_out/diff_launch.log 2>&1
