#!/bin/bash
# Round-end evidence in one gpurun job: GPU parity suite, smoke, bench lines for every config,
# and the cfg2 ncu launch list of the default bench command.
# usage (from this container): gpurun --timeout 3000 -- 'bash tools/gpu_round.sh r01v3'
TAG=${1:-r01}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_$TAG.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.txt 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.txt 2>&1
echo "smoke exit $?" >> gpurun_out/smoke_$TAG.txt
for c in cfg2 cfg2b1 cfg1 cfg4 cfg3 cfg3k cfg5; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 3 > gpurun_out/bench_${c}_$TAG.json 2> gpurun_out/bench_${c}_$TAG.err
  echo "bench $c exit $?" >> gpurun_out/bench_${c}_$TAG.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_cfg2_ref_$TAG.json 2> gpurun_out/bench_cfg2_ref_$TAG.err
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"seg_gemm|gather_blocked|sym_pass|csr_sum" -c 400 --csv --log-file gpurun_out/launches_bench_cfg2_$TAG.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench_$TAG.log 2>&1
tail -n 2 gpurun_out/pytest_gpu_$TAG.txt gpurun_out/smoke_$TAG.txt
for c in cfg2 cfg2b1 cfg1 cfg4 cfg3 cfg3k cfg5; do python -c "
import json,sys
try:
    d=json.loads(open('gpurun_out/bench_${c}_$TAG.json').read().strip().splitlines()[-1]); print('$c', d.get('value'), d.get('unit'), d.get('ms_per_step'))
except Exception as e: print('$c', 'ERR', e)"; done
