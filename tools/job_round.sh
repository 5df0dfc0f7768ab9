bash tools/gpu_round.sh r01v11
timeout 900 python bench.py > gpurun_out/bench_default_r01v11.json 2> gpurun_out/bench_default_r01v11.err
echo "default bench exit $?" >> gpurun_out/bench_default_r01v11.err
