"""A/B of the stage-5 split (h2b_tune 9) on cfg2: ms per hgemv at several b."""
import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2003_10173_b200 import H2Matrix, build_block_tree, build_cluster_tree
from paper_2003_10173_b200._lib import lib, check
import bench
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
c = bench.CONFIGS[cfg]
pts = bench.grid_points(c["grid"])
n = pts.shape[0]
ct = build_cluster_tree(pts, c["leaf"], device=True)
bt = build_block_tree(ct, ct, 1.0)
m = H2Matrix.kernel(bt, pts, c["kind"], c["ell"], c["rank"])
s = torch.cuda.current_stream().cuda_stream
for b in [int(v) for v in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["32", "16", "4"])]:
    X = torch.randn(b, n, dtype=torch.float64, device="cuda")
    res = {}
    ys = {}
    for knob in (0, 1, 0, 1):
        lib.h2b_tune(9, knob)
        Y = torch.empty_like(X)
        for _ in range(4):
            check(lib.h2c_hgemv(m._h, 0, 0, n, b, X.data_ptr(), n, Y.data_ptr(), n, 1.0, 0.0, s))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            check(lib.h2c_hgemv(m._h, 0, 0, n, b, X.data_ptr(), n, Y.data_ptr(), n, 1.0, 0.0, s))
        e1.record(); torch.cuda.synchronize()
        res.setdefault(knob, []).append(e0.elapsed_time(e1) / 20)
        ys[knob] = Y.clone()
    d = float((ys[0] - ys[1]).abs().max() / ys[0].abs().max())
    print(f"{cfg} b={b}: split off {min(res[0]):.4f} ms, split on {min(res[1]):.4f} ms, rel diff {d:.2e}", flush=True)
lib.h2b_tune(9, 1)
