"""Per-launch CUDA-event times of one hgemv (stage id, ms) for a bench config."""
import argparse
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2003_10173_b200 import H2Matrix, build_block_tree, build_cluster_tree  # noqa: E402
from paper_2003_10173_b200._lib import check, lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2b1")
a = ap.parse_args()
cfg = bench.CONFIGS[a.config]
b = cfg["b"]
pts = bench.grid_points(cfg["grid"])
n = pts.shape[0]
ct = build_cluster_tree(pts, cfg["leaf"])
bt = build_block_tree(ct, ct, 1.0)
m = H2Matrix.kernel(bt, pts, cfg["kind"], cfg["ell"], cfg["rank"])
x = torch.randn(b, n, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
maxrec = 256
cnt = C.c_int()
st = np.zeros(maxrec, np.int32)
ms = np.zeros(maxrec)
sh = torch.cuda.current_stream().cuda_stream
acc = None
for r in range(6):
    check(lib.h2c_hgemv_stage_times(m._h, 0, 0, n, b, x.data_ptr(), n, y.data_ptr(), n, sh, maxrec, C.byref(cnt),
                                    st.ctypes.data_as(C.c_void_p), ms.ctypes.data_as(C.c_void_p), None, None))
    if r == 0:
        continue
    acc = ms[:cnt.value].copy() if acc is None else acc + ms[:cnt.value]
acc /= 5
for i in range(cnt.value):
    print(f"launch {i:2d} stage {st[i]} {acc[i]*1e3:8.1f} us")
print(f"total {acc.sum():.3f} ms")
