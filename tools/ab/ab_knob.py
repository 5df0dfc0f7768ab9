"""Generic A/B of one h2b_tune knob: ab_knob.py cfg b_list which v1,v2,... (ms per hgemv, bitwise check)."""
import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2003_10173_b200 import H2Matrix, build_block_tree, build_cluster_tree
from paper_2003_10173_b200._lib import lib, check
import bench
cfg, bl, which = sys.argv[1], [int(v) for v in sys.argv[2].split(",")], int(sys.argv[3])
vals = [int(v) for v in sys.argv[4].split(",")]
c = bench.CONFIGS[cfg]
pts = bench.grid_points(c["grid"]); n = pts.shape[0]
ct = build_cluster_tree(pts, c["leaf"], device=True); bt = build_block_tree(ct, ct, 1.0)
m = H2Matrix.kernel(bt, pts, c["kind"], c["ell"], c["rank"])
s = torch.cuda.current_stream().cuda_stream
for b in bl:
    X = torch.randn(b, n, dtype=torch.float64, device="cuda")
    res, ys = {}, {}
    for v in vals + vals + vals:
        lib.h2b_tune(which, v)
        Y = torch.empty_like(X)
        for _ in range(4):
            check(lib.h2c_hgemv(m._h, 0, 0, n, b, X.data_ptr(), n, Y.data_ptr(), n, 1.0, 0.0, s))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            check(lib.h2c_hgemv(m._h, 0, 0, n, b, X.data_ptr(), n, Y.data_ptr(), n, 1.0, 0.0, s))
        e1.record(); torch.cuda.synchronize()
        res.setdefault(v, []).append(e0.elapsed_time(e1) / 20)
        ys[v] = Y.clone()
    same = all(torch.equal(ys[k], ys[vals[0]]) for k in ys)
    print(f"{cfg} b={b} knob{which}: " + " ".join(f"{k}={min(t):.4f}/{max(t):.4f}" for k, t in res.items()) + f" ms (min/max of 3); bitwise {same}", flush=True)
