"""Minimal driver for ncu: build one bench configuration, run `--reps` hgemvs.

  python tools/prof_hgemv.py [--config cfg2] [--b 32] [--reps 2]
Kernel launch order of one hgemv (transpose=0): gather, leaf upsweep, transfer
upsweep per level, coupling, downsweep per level, leaf + dense near-field.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2003_10173_b200 import H2Matrix, build_block_tree, build_cluster_tree  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2", choices=list(bench.CONFIGS))
    ap.add_argument("--b", type=int, default=0)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--tune", default="", help="h2b_tune values for slots 0,1,2 (e.g. 0,0,2)")
    a = ap.parse_args()
    if a.tune:
        import ctypes as C
        from paper_2003_10173_b200._lib import lib
        lib.h2b_tune.argtypes = [C.c_int, C.c_int]
        for i, v in enumerate(a.tune.split(",")):
            lib.h2b_tune(i, int(v))
    cfg = bench.CONFIGS[a.config]
    b = a.b or cfg["b"]
    pts = bench.grid_points(cfg["grid"])
    n = pts.shape[0]
    ct = build_cluster_tree(pts, cfg["leaf"])
    bt = build_block_tree(ct, ct, 1.0)
    m = H2Matrix.kernel(bt, pts, cfg["kind"], cfg["ell"], cfg["rank"])
    x = torch.randn(b, n, dtype=torch.float64, device="cuda").t()
    y = torch.empty(b, n, dtype=torch.float64, device="cuda").t()
    for _ in range(a.reps):
        m.hgemv(x, y)
    torch.cuda.synchronize()
    print(f"ok {a.config} n={n} b={b} launches/hgemv={m.launches(b)} |y|={float(y.norm()):.6e}")


if __name__ == "__main__":
    main()
