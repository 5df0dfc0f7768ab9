export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_diffusion_gpu.py -x -q > gpurun_out/pytest_diff.txt 2>&1; echo "exit $?" >> gpurun_out/pytest_diff.txt
timeout 300 python tools/diff1d_probe.py --b 1 3 16 64 --check 2 > gpurun_out/diff_probe.txt 2>&1
