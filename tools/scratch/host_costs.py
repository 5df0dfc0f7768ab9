import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2003_10173_b200 import *
from paper_2003_10173_b200._lib import lib, check
import bench
pts = bench.grid_points((262144,))
ct = build_cluster_tree(pts, 32); bt = build_block_tree(ct, ct, 1.0, Admissibility.weak)
m = H2Matrix.kernel(bt, pts, "gaussian", 0.05, 16)
n = pts.shape[0]
X = torch.randn(16, n, dtype=torch.float64, device="cuda"); Y = torch.empty_like(X)
s = torch.cuda.current_stream().cuda_stream
def T(f, k=5):
    f(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(k): f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / k * 1e3
print("hgemv b16 (plan cached) ms", T(lambda: check(lib.h2c_hgemv(m._h, 0, 0, n, 16, X.data_ptr(), n, Y.data_ptr(), n, 1.0, 0.0, s))))
print("orthogonalize ms", T(lambda: orthogonalize(m)))
g = orthogonalize(m)
print("recompress(orth) ms", T(lambda: recompress(g, 1e-7)))
print("recompress(raw) ms", T(lambda: recompress(m, 1e-7)))
def newplan():
    mm = H2Matrix.kernel(bt, pts, "gaussian", 0.05, 16)
    torch.cuda.synchronize()
    t = time.perf_counter()
    check(lib.h2c_hgemv(mm._h, 0, 0, n, 16, X.data_ptr(), n, Y.data_ptr(), n, 1.0, 0.0, s))
    torch.cuda.synchronize()
    return (time.perf_counter() - t) * 1e3
print("hgemv incl plan build ms", [round(newplan(), 2) for _ in range(3)])
