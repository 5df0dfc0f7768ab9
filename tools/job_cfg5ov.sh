# cfg5 with the few-vector dense overlap off / on (h2b_tune 8), alternating, to separate the effect from box noise
mkdir -p gpurun_out
for o in 0 1 0 1; do
timeout 600 python -c "
import sys, ctypes as C
sys.argv=['bench.py','--config','cfg5','--steps','2','--warmup','1']
from paper_2003_10173_b200._lib import lib
lib.h2b_tune.argtypes=[C.c_int,C.c_int]; lib.h2b_tune(8,$o)
import bench; bench.main()" > gpurun_out/cfg5ov_$o.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/cfg5ov_$o.json').read().strip().splitlines()[-1]); print('overlap $o', d['value'], [r[4] for r in d['inversion']['rows']])" >> gpurun_out/cfg5ov.txt
done
cat gpurun_out/cfg5ov.txt
