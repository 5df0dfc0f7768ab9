"""Task / entry order sweep of the b >= 16 hgemv plans (GPU).

  python tools/order_probe.py [--config cfg2] [--combos 0:0,1:0,1:1] [--reps 10]

Each combo "e:t[:f]" sets h2b_tune(5, e) (entry order inside a task) and h2b_tune(6, t)
(task order inside a launch), h2b_tune(7, f) (programmatic dependent launch), h2b_tune(8, o)
(few-vector path: dense pass concurrent with the sweeps), builds a fresh matrix (plans are cached per matrix),
and prints per-stage CUDA-event times plus the whole-hgemv time of CUDA-graph
replays. Every combo is checked against the first one (round-off only).
Run under ncu with --kernel-name regex to read the DRAM bytes per combo.
"""
import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2003_10173_b200 import H2Matrix, build_block_tree, build_cluster_tree  # noqa: E402
from paper_2003_10173_b200._lib import lib  # noqa: E402
from tune_hgemv import stage_times  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2", choices=list(bench.CONFIGS))
    ap.add_argument("--combos", default="0:0,1:0,1:1,0:1")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--no-stages", action="store_true")
    a = ap.parse_args()
    lib.h2b_tune.argtypes = [C.c_int, C.c_int]
    lib.h2b_tune.restype = C.c_int
    cfg = bench.CONFIGS[a.config]
    b = cfg["b"]
    pts = bench.grid_points(cfg["grid"])
    n = pts.shape[0]
    ct = build_cluster_tree(pts, cfg["leaf"])
    bt = build_block_tree(ct, ct, 1.0)
    x = torch.randn(b, n, dtype=torch.float64, device="cuda").t()
    y = torch.empty(b, n, dtype=torch.float64, device="cuda").t()
    y0 = None
    for combo in a.combos.split(","):
        e, t, f, o = (list(int(q) for q in combo.split(":")) + [1, 1])[:4]
        lib.h2b_tune(8, o)
        lib.h2b_tune(5, e)
        lib.h2b_tune(6, t)
        lib.h2b_tune(7, f)
        m = H2Matrix.kernel(bt, pts, cfg["kind"], cfg["ell"], cfg["rank"])
        m.hgemv(x, y)
        torch.cuda.synchronize()
        if y0 is None:
            y0 = y.clone()
        diff = float((y - y0).abs().max() / y0.abs().max())
        line = ""
        if not a.no_stages:
            agg = stage_times(m, x, y, n, b, 3)
            line = " ".join(f"s{k}={agg[k][0]:.3f}" for k in sorted(agg))
        for _ in range(3):
            m.hgemv(x, y)
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s0.record()
        for _ in range(a.reps):
            m.hgemv(x, y)
        s1.record()
        torch.cuda.synchronize()
        ms = s0.elapsed_time(s1) / a.reps
        print(f"entry {e} task {t} pdl {f} overlap {o}: hgemv {ms:.3f} ms  {line}  maxdiff {diff:.1e}", flush=True)
        del m
    lib.h2b_tune(5, 1)
    lib.h2b_tune(6, 0)
    lib.h2b_tune(7, 1)
    lib.h2b_tune(8, 1)


if __name__ == "__main__":
    main()
