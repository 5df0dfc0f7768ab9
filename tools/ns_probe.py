"""cfg5 on the minimal-surface Hessian (surface<N>): HARA of the sparse black box,
regularisation alpha I, then recompress + rank-8 update + hierarchical
Newton-Schulz, for a list of shifts. Prints iterations, residuals and times.

  python tools/ns_probe.py [--grid 256] [--alpha 1.0 0.3 0.1]
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2003_10173_b200 import (PeelConfig, ThresholdSchedule, build_block_tree, build_cluster_tree,  # noqa: E402
                                   h_newton_schulz, low_rank_update, make_oracle, peel_construct, recompress,
                                   residual_norm, scaled_identity_start)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=256)
    ap.add_argument("--alpha", type=float, nargs="+", default=[1.0, 0.3, 0.1])
    ap.add_argument("--eps", type=float, default=1e-6)
    a = ap.parse_args()
    torch.cuda.init()
    o = make_oracle(f"surface{a.grid}")
    ct = build_cluster_tree(o.points, o.leaf)
    bt = build_block_tree(ct, ct, o.eta, o.mode)
    t0 = time.perf_counter()
    h = peel_construct(o.op, bt, PeelConfig(eps=1e-8, rng=1))
    torch.cuda.synchronize()
    print(f"HARA of surface{a.grid}: {time.perf_counter() - t0:.3f} s, {h.stats.total} samples, "
          f"ranks {h.matrix.rank_profile()}", flush=True)
    n = o.op.dim()
    X = 0.1 * np.random.default_rng(7).standard_normal((n, 8))
    for alpha in a.alpha:
        m = recompress(h.matrix, 1e-12)
        m.add_diagonal(alpha)
        t0 = time.perf_counter()
        ar = recompress(m, 1e-8)
        au = low_rank_update(ar, X, X, 1e-8)
        x0 = scaled_identity_start(au)
        try:
            res = h_newton_schulz(au, x0, ThresholdSchedule(dynamic=True), a.eps, PeelConfig(eps=a.eps, rng=1))
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            rows = [(r.iter, f"{r.residual:.2e}", f"{r.eps_k:.1e}", r.samples) for r in res.trace.rows]
            print(f"alpha {alpha}: {dt:.3f} s, {len(rows)} iterations, final {res.trace.final_residual:.2e}, "
                  f"check {residual_norm(au, res.X):.2e}, ranks {res.X.rank_profile()}\n   {rows}", flush=True)
        except Exception as e:
            tr = getattr(e, "trace", None)
            rows = [(r.iter, f"{r.residual:.2e}") for r in tr.rows] if tr else []
            print(f"alpha {alpha}: FAILED {e} {rows}", flush=True)


if __name__ == "__main__":
    main()
