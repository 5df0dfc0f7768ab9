"""Run one config's hgemv a few times (for ncu launch lists / captures): run_cfg.py cfg b reps"""
import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2003_10173_b200 import H2Matrix, build_block_tree, build_cluster_tree
from paper_2003_10173_b200._lib import lib, check
import bench
c = bench.CONFIGS[sys.argv[1]]; b = int(sys.argv[2])
pts = bench.grid_points(c["grid"]); n = pts.shape[0]
ct = build_cluster_tree(pts, c["leaf"], device=True); bt = build_block_tree(ct, ct, 1.0)
m = H2Matrix.kernel(bt, pts, c["kind"], c["ell"], c["rank"])
X = torch.randn(b, n, dtype=torch.float64, device="cuda"); Y = torch.empty_like(X)
s = torch.cuda.current_stream().cuda_stream
print("launches per hgemv:", m.launches(b), flush=True)
for _ in range(int(sys.argv[3])):
    check(lib.h2c_hgemv(m._h, 0, 0, n, b, X.data_ptr(), n, Y.data_ptr(), n, 1.0, 0.0, s))
torch.cuda.synchronize()
