bash tools/gpu_round.sh r01v8
timeout 900 python bench.py > gpurun_out/bench_default_r01v8.json 2> gpurun_out/bench_default_r01v8.err
echo "default bench exit $?" >> gpurun_out/bench_default_r01v8.err
bash tools/gpu_prof.sh cfg2 r01v8 seg_gemm_kernelILi64ELi32ELi2ELi2ELi2ELi32ELb1ELi2E seg_gemm_kernelILi32ELi32ELi2ELi2ELi1ELi32ELb1ELi0E 15
