mkdir -p gpurun_out
LD_PRELOAD=tools/sprof.so SPROF_OUT=gpurun_out/sprof_cfg3k.txt timeout 600 python bench.py --config cfg3k --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/hara_cfg3k.json 2> gpurun_out/hara_cfg3k.err
