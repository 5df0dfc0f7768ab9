"""HARA on the device diffusion Hessian (cfg3 faithful form): build time split
into operator and construction time, samples, rank profile, accuracy."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2003_10173_b200 import PeelConfig, estimate_relative_error, make_oracle, peel_construct


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=262144)
    ap.add_argument("--steps", type=int, default=64)
    ap.add_argument("--eps", type=float, default=1e-6)
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    t = time.perf_counter()
    o = make_oracle(f"diff1d-{a.n}", {"steps": str(a.steps)})
    bt = o.default_block_tree()
    torch.cuda.synchronize()
    print(f"setup {time.perf_counter() - t:.2f} s")
    for r in range(a.reps):
        o.op.reset_counter()
        t = time.perf_counter()
        res = peel_construct(o.op, bt, PeelConfig(eps=a.eps, rng=1))
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        print(f"build {dt:.3f} s  op {res.op_ms / 1e3:.3f} s  samples {res.stats.total}  "
              f"cols {o.op.columns_applied()}")
    print("levels", [(lv.level, lv.max_rank, lv.samples) for lv in res.stats.levels])
    print("rank profile", list(res.matrix.rank_profile()))
    t = time.perf_counter()
    print("estimated relative error", estimate_relative_error(o.op, res.matrix), f"({time.perf_counter() - t:.2f} s)")


if __name__ == "__main__":
    main()
