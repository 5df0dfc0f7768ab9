bash tools/gpu_round.sh r01v7
timeout 900 python bench.py > gpurun_out/bench_default_r01v7.json 2> gpurun_out/bench_default_r01v7.err
echo "default bench exit $?" >> gpurun_out/bench_default_r01v7.err
