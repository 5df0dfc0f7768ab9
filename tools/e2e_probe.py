"""Probe: device, synchronous and pipelined host-buffer hgemv with / without graph replay."""
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2003_10173_b200 import H2Matrix, build_block_tree, build_cluster_tree  # noqa: E402
from paper_2003_10173_b200._lib import check, lib  # noqa: E402

lib.h2b_tune.argtypes = [C.c_int, C.c_int]
cfg = bench.CONFIGS["cfg2"]
pts = bench.grid_points(cfg["grid"])
n, b = pts.shape[0], 32
ct = build_cluster_tree(pts, 64)
bt = build_block_tree(ct, ct, 1.0)
m = H2Matrix.kernel(bt, pts, "gaussian", 0.1, 32)
xp = torch.randn(b, n, dtype=torch.float64).pin_memory()
yps = [torch.empty(b, n, dtype=torch.float64).pin_memory() for _ in range(3)]
X = xp.cuda()
Y = torch.empty_like(X)
streams = [torch.cuda.Stream() for _ in range(3)]
# KNOB=which VALS=v1,v2 (default: graph replay off / on)
knob = int(os.environ.get("KNOB", "3"))
vals = [int(v) for v in os.environ.get("VALS", "0,1").split(",")]
for graph in vals + vals:
    lib.h2b_tune(knob, graph)
    for _ in range(3):
        check(lib.h2c_hgemv(m._h, 0, 0, n, b, X.data_ptr(), n, Y.data_ptr(), n, 1.0, 0.0, None))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        check(lib.h2c_hgemv(m._h, 0, 0, n, b, X.data_ptr(), n, Y.data_ptr(), n, 1.0, 0.0, None))
    torch.cuda.synchronize()
    td = (time.perf_counter() - t0) / 10
    for _ in range(3):
        check(lib.h2c_matvec_host(m._h, 0, 0, n, b, xp.data_ptr(), yps[0].data_ptr()))
    t0 = time.perf_counter()
    for _ in range(5):
        check(lib.h2c_matvec_host(m._h, 0, 0, n, b, xp.data_ptr(), yps[0].data_ptr()))
    ts = (time.perf_counter() - t0) / 5
    for i in range(6):
        check(lib.h2c_matvec_host_async(m._h, 0, 0, n, b, xp.data_ptr(), yps[i % 3].data_ptr(),
                                        streams[i % 3].cuda_stream))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(12):
        check(lib.h2c_matvec_host_async(m._h, 0, 0, n, b, xp.data_ptr(), yps[i % 3].data_ptr(),
                                        streams[i % 3].cuda_stream))
    torch.cuda.synchronize()
    ta = (time.perf_counter() - t0) / 12
    t0 = time.perf_counter()
    for _ in range(5):
        X.copy_(xp, non_blocking=True)
    torch.cuda.synchronize()
    th = (time.perf_counter() - t0) / 5
    t0 = time.perf_counter()
    for _ in range(5):
        yps[0].copy_(X, non_blocking=True)
    torch.cuda.synchronize()
    tdh = (time.perf_counter() - t0) / 5
    print(f"knob{knob}={graph}: device {td*1e3:.2f} ms, sync host {ts*1e3:.2f} ms, async3 {ta*1e3:.2f} ms, "
          f"H2D {th*1e3:.2f} ms ({8*n*b/th/1e9:.1f} GB/s), D2H {tdh*1e3:.2f} ms ({8*n*b/tdh/1e9:.1f} GB/s)",
          flush=True)
