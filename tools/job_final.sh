# final-state evidence: full GPU suite, smoke, default bench line, few-vector configs
TAG=${1:-r01v12}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.txt 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.txt 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_$TAG.txt
timeout 900 python bench.py > gpurun_out/bench_default_$TAG.json 2> gpurun_out/bench_default_$TAG.err
for c in cfg1 cfg2b1; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 > gpurun_out/bench_${c}_$TAG.json 2>/dev/null; done
tail -n 2 gpurun_out/pytest_gpu_$TAG.txt gpurun_out/smoke_$TAG.txt
for c in default cfg1 cfg2b1; do python -c "
import json; d=json.loads(open('gpurun_out/bench_${c}_$TAG.json').read().strip().splitlines()[-1]); print('$c', d['value'], d['unit'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['clocks'])"; done
