#!/bin/bash
# One gpurun job: FP64 peak, GPU parity tests, smoke, a short bench line.
# usage (from this container): gpurun --timeout 1500 -- 'bash tools/gpu_check.sh'
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
nproc > gpurun_out/nproc.txt; lscpu | head -20 >> gpurun_out/nproc.txt
[ -x tools/fp64_peak ] && timeout 120 tools/fp64_peak > gpurun_out/fp64_peak.txt 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
echo "smoke exit $?" >> gpurun_out/smoke.txt
timeout 600 python bench.py --steps 10 --warmup 3 ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench exit $?" >> gpurun_out/bench.err
tail -n 3 gpurun_out/pytest_gpu.txt gpurun_out/smoke.txt gpurun_out/bench.err
