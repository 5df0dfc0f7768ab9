"""cfg2 b=1: dense overlap (h2b_tune 8) on/off x TMA (h2b_tune 10) on/off: ms per hgemv."""
import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2003_10173_b200 import H2Matrix, build_block_tree, build_cluster_tree
from paper_2003_10173_b200._lib import lib, check
import bench
c = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]
pts = bench.grid_points(c["grid"]); n = pts.shape[0]
ct = build_cluster_tree(pts, c["leaf"], device=True); bt = build_block_tree(ct, ct, 1.0)
m = H2Matrix.kernel(bt, pts, c["kind"], c["ell"], c["rank"])
s = torch.cuda.current_stream().cuda_stream
X = torch.randn(1, n, dtype=torch.float64, device="cuda")
res = {}
for rep in range(2):
    for ov in (1, 0):
        for tma in (1, 0):
            lib.h2b_tune(8, ov); lib.h2b_tune(10, tma)
            Y = torch.empty_like(X)
            for _ in range(4):
                check(lib.h2c_hgemv(m._h, 0, 0, n, 1, X.data_ptr(), n, Y.data_ptr(), n, 1.0, 0.0, s))
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                check(lib.h2c_hgemv(m._h, 0, 0, n, 1, X.data_ptr(), n, Y.data_ptr(), n, 1.0, 0.0, s))
            e1.record(); torch.cuda.synchronize()
            res.setdefault((ov, tma), []).append(e0.elapsed_time(e1) / 20)
for k, v in res.items():
    print(f"overlap={k[0]} tma={k[1]}: {min(v):.4f} ms")
lib.h2b_tune(8, 1); lib.h2b_tune(10, 1)
