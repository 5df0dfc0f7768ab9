"""Per-launch device times (h2c_hgemv_stage_times, serialised) for one config and b."""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch, ctypes as C
from paper_2003_10173_b200 import H2Matrix, build_block_tree, build_cluster_tree
from paper_2003_10173_b200._lib import lib, check
import bench
cfg = bench.CONFIGS[sys.argv[1]]
b = int(sys.argv[2])
pts = bench.grid_points(cfg["grid"]); n = pts.shape[0]
ct = build_cluster_tree(pts, cfg["leaf"], device=True); bt = build_block_tree(ct, ct, 1.0)
m = H2Matrix.kernel(bt, pts, cfg["kind"], cfg["ell"], cfg["rank"])
X = torch.randn(b, n, dtype=torch.float64, device="cuda"); Y = torch.empty_like(X)
s = torch.cuda.current_stream().cuda_stream
cnt = C.c_int(); st = np.zeros(512, np.int32); ms = np.zeros(512); fl = np.zeros(512); by = np.zeros(512)
best = None
for rep in range(6):
    check(lib.h2c_hgemv_stage_times(m._h, 0, 0, n, b, X.data_ptr(), n, Y.data_ptr(), n, s, 512, C.byref(cnt),
          st.ctypes.data_as(C.c_void_p), ms.ctypes.data_as(C.c_void_p), fl.ctypes.data_as(C.c_void_p), by.ctypes.data_as(C.c_void_p)))
    cur = ms[:cnt.value].copy()
    best = cur if best is None else np.minimum(best, cur)
print(f"{sys.argv[1]} b={b}: {cnt.value} launches, sum {best.sum():.4f} ms")
for i in range(cnt.value):
    print(f"  {i:3d} stage {st[i]}  {best[i]*1e3:8.1f} us  {fl[i]*b/1e6:9.2f} MF  {by[i]/1e6:8.2f} MB")
