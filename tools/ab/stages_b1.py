import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch, ctypes as C
from paper_2003_10173_b200 import H2Matrix, build_block_tree, build_cluster_tree
from paper_2003_10173_b200._lib import lib, check
import bench
cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2b1"]
pts = bench.grid_points(cfg["grid"]); n = pts.shape[0]
ct = build_cluster_tree(pts, cfg["leaf"], device=True); bt = build_block_tree(ct, ct, 1.0)
m = H2Matrix.kernel(bt, pts, cfg["kind"], cfg["ell"], cfg["rank"])
b = int(sys.argv[2]) if len(sys.argv) > 2 else 1
X = torch.randn(b, n, dtype=torch.float64, device="cuda"); Y = torch.empty_like(X)
s = torch.cuda.current_stream().cuda_stream
for knob in (0, 1):
    lib.h2b_tune(10, knob)
    cnt = C.c_int(); st = np.zeros(256, np.int32); ms = np.zeros(256); fl = np.zeros(256); by = np.zeros(256)
    for rep in range(4):
        check(lib.h2c_hgemv_stage_times(m._h, 0, 0, n, b, X.data_ptr(), n, Y.data_ptr(), n, s, 256, C.byref(cnt),
              st.ctypes.data_as(C.c_void_p), ms.ctypes.data_as(C.c_void_p), fl.ctypes.data_as(C.c_void_p), by.ctypes.data_as(C.c_void_p)))
    recs = [(int(st[i]), round(float(ms[i]), 4), round(by[i] / 1e9, 3)) for i in range(cnt.value)]
    tot = sum(r[1] for r in recs)
    print("tma", knob, "sum", round(tot, 4), "ms;", [r for r in recs if r[1] > 0.02])
