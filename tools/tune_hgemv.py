"""Tile-shape sweep of the b >= 32 seg_gemm instances on one config (GPU).

  python tools/tune_hgemv.py [--config cfg2] [--reps 5]
Prints per-stage CUDA-event times for each variant and checks every variant
against variant 0 (the results must agree to round-off).
"""
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


def stage_times(m, x, y, n, b, reps):
    maxrec = 256
    cnt = C.c_int()
    st = np.zeros(maxrec, np.int32)
    ms = np.zeros(maxrec)
    fl = np.zeros(maxrec)
    by = np.zeros(maxrec)
    agg = {}
    sh = torch.cuda.current_stream().cuda_stream
    for r in range(reps + 1):
        check(lib.h2c_hgemv_stage_times(m._h, 0, 0, n, b, x.data_ptr(), n, y.data_ptr(), n, sh, maxrec,
                                        C.byref(cnt), st.ctypes.data_as(C.c_void_p), ms.ctypes.data_as(C.c_void_p),
                                        fl.ctypes.data_as(C.c_void_p), by.ctypes.data_as(C.c_void_p)))
        if r == 0:
            continue
        for i in range(cnt.value):
            a = agg.setdefault(int(st[i]), [0.0, 0.0])
            a[0] += ms[i] / reps
            a[1] += fl[i] / reps
    return agg


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2", choices=list(bench.CONFIGS))
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--dense", default="0,1")
    ap.add_argument("--coupling", default="0,1")
    ap.add_argument("--ws", default="", help="warp-specialised kernel variants (h2b_tune(2, v)); 0 = off")
    a = ap.parse_args()
    lib.h2b_tune.argtypes = [C.c_int, C.c_int]
    lib.h2b_tune.restype = C.c_int
    cfg = bench.CONFIGS[a.config]
    b = cfg["b"]
    pts = bench.grid_points(cfg["grid"])
    n = pts.shape[0]
    ct = build_cluster_tree(pts, cfg["leaf"])
    bt = build_block_tree(ct, ct, 1.0)
    m = H2Matrix.kernel(bt, pts, cfg["kind"], cfg["ell"], cfg["rank"])
    x = torch.randn(b, n, dtype=torch.float64, device="cuda").t()
    y = torch.empty(b, n, dtype=torch.float64, device="cuda").t()
    lib.h2b_tune(0, 0)
    lib.h2b_tune(1, 0)
    lib.h2b_tune(2, 0)
    m.hgemv(x, y)
    y0 = y.clone()
    for v in [int(q) for q in a.ws.split(",") if q]:
        lib.h2b_tune(2, v)
        m.hgemv(x, y)
        torch.cuda.synchronize()
        diff = float((y - y0).abs().max() / y0.abs().max())
        agg = stage_times(m, x, y, n, b, a.reps)
        tot = sum(s_[0] for s_ in agg.values())
        line = " ".join(f"s{k}={agg[k][0]:.3f}ms({agg[k][1] / agg[k][0] / 1e9:.1f}TF)" for k in sorted(agg)
                        if agg[k][1] > 0)
        print(f"ws v{v}: total {tot:.3f} ms  {line}  maxdiff {diff:.1e}", flush=True)
    lib.h2b_tune(2, 0)
    for which, vals in ((0, a.dense), (1, a.coupling)):
        for v in [int(s) for s in vals.split(",")]:
            lib.h2b_tune(0, 0)
            lib.h2b_tune(1, 0)
            lib.h2b_tune(which, v)
            m.hgemv(x, y)
            torch.cuda.synchronize()
            diff = float((y - y0).abs().max() / y0.abs().max())
            agg = stage_times(m, x, y, n, b, a.reps)
            tot = sum(s[0] for s in agg.values())
            line = " ".join(f"s{k}={agg[k][0]:.3f}ms({agg[k][1] / agg[k][0] / 1e9:.1f}TF)" for k in sorted(agg)
                            if agg[k][1] > 0)
            print(f"{'dense' if which == 0 else 'coupl'} v{v}: total {tot:.3f} ms  {line}  maxdiff {diff:.1e}",
                  flush=True)
    lib.h2b_tune(0, 0)
    lib.h2b_tune(1, 0)


if __name__ == "__main__":
    main()
