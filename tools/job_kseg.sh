export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_diffusion_gpu.py -x -q > gpurun_out/pytest_kseg.txt 2>&1; echo "exit $?" >> gpurun_out/pytest_kseg.txt
timeout 300 python tools/diff1d_probe.py --b 16 64 --check 0 > gpurun_out/diff_probe_kseg.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"carry" --csv --log-file gpurun_out/kseg_launches.csv python tools/diff1d_probe.py --b 16 --reps 1 --check 0 > /dev/null 2>&1
