"""The NS testbed matrix of cfg5 (surface<N> Hessian, HARA at eps 1e-8, + alpha I,
recompress, rank-8 update) built on the B200, exported for the reference's own
inversion driver (oracle/_ref, run on the CPU), plus the B200's NS trace on it.

  python tools/ns_testbed.py --grid 64 --out gpurun_out/ns_surface64.npz     (GPU box)
  python tools/ns_testbed.py --reference gpurun_out/ns_surface64.npz         (CPU: the reference's NS)
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def build(a):
    import torch
    from paper_2003_10173_b200 import (PeelConfig, ThresholdSchedule, build_block_tree, build_cluster_tree,
                                       h_newton_schulz, low_rank_update, make_oracle, peel_construct, recompress,
                                       residual_norm, scaled_identity_start)
    o = make_oracle(f"surface{a.grid}")
    ct = build_cluster_tree(o.points, o.leaf)
    bt = build_block_tree(ct, ct, o.eta, o.mode)
    h = peel_construct(o.op, bt, PeelConfig(eps=1e-8, rng=0))
    n = o.op.dim()
    X = 0.1 * np.random.default_rng(7).standard_normal((n, 8))
    m = recompress(h.matrix, 1e-12)
    m.add_diagonal(a.alpha)
    ar = recompress(m, 1e-8)
    au = low_rank_update(ar, X, X, 1e-8)
    rr, cr = au.ranks()
    parts = au.download()
    out = {"points": np.asarray(o.points), "leaf": o.leaf, "eta": o.eta, "strong": int(o.mode == 0),
           "ranks": rr, "alpha": a.alpha}
    out.update({f"part_{k}": v for k, v in parts.items()})
    x0 = scaled_identity_start(au)
    t0 = time.perf_counter()
    try:
        res = h_newton_schulz(au, x0, ThresholdSchedule(dynamic=True), a.eps, PeelConfig(eps=a.eps, rng=0))
        rows = [(r.iter, r.residual, r.eps_k, r.samples) for r in res.trace.rows]
        final, conv = res.trace.final_residual, res.trace.converged
    except Exception as e:
        tr = getattr(e, "trace", None)
        rows = [(r.iter, r.residual, r.eps_k, r.samples) for r in tr.rows] if tr else []
        final, conv = float("nan"), False
    torch.cuda.synchronize()
    out["b200_trace"] = np.array(rows, dtype=float)
    out["b200_seconds"] = time.perf_counter() - t0
    out["b200_converged"] = int(conv)
    out["b200_final"] = final
    np.savez_compressed(a.out, **out)
    print(json.dumps({"n": n, "converged": conv, "final": final, "iters": len(rows),
                      "seconds": out["b200_seconds"], "trace": [[int(r[0]), f"{r[1]:.2e}", r[2], int(r[3])] for r in rows]}))


def reference(a):
    from oracle import pyref as R
    d = np.load(a.reference)
    tree = R.Tree(d["points"], int(d["leaf"]), float(d["eta"]), not bool(d["strong"]))
    parts = {k[5:]: d[k] for k in d.files if k.startswith("part_")}
    h = R.H2.from_packed(tree, True, d["ranks"], None, parts)
    t0 = time.perf_counter()
    x, rows, final, conv = h.h_inverse(a.eps, dynamic=True)
    dt = time.perf_counter() - t0
    print(json.dumps({"reference_converged": conv, "final": final, "iters": len(rows), "seconds": dt,
                      "trace": [[int(r[0]), f"{r[1]:.2e}", r[2], int(r[3])] for r in rows],
                      "b200_trace": [[int(r[0]), f"{r[1]:.2e}", r[2], int(r[3])] for r in d["b200_trace"]],
                      "b200_converged": int(d["b200_converged"])}))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=64)
    ap.add_argument("--alpha", type=float, default=1.0)
    ap.add_argument("--eps", type=float, default=1e-6)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "ns_testbed.npz"))
    ap.add_argument("--reference", default=None)
    a = ap.parse_args()
    reference(a) if a.reference else build(a)
