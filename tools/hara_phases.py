"""Host wall-time breakdown of one HARA build without stream draining
(h2b_hara_phase_sync(0)): each phase's time is the host time spent in it,
including any blocking it does (the per-panel singular-value read back, the
truncation rank read back, plan builds). Compare with the drained split that
bench.py reports as phases_s.

  python tools/hara_phases.py [--config cfg3k] [--reps 3]
"""
import argparse
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2003_10173_b200 import PeelConfig, peel_construct  # noqa: E402
from paper_2003_10173_b200._lib import lib  # noqa: E402

NAMES = ["rng", "op_apply", "residual_hgemv", "absorb", "transposed_pass", "local_updates", "recompress",
         "dense_leaves", "orthogonalize", "truncation_bases", "projection"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3k")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    cfg = bench.CONFIGS[a.config]
    n = cfg["grid"][0]
    op, bt, keep = bench.hara_operator(cfg, n)
    pc = PeelConfig(eps=cfg["eps"], rng=1)
    peel_construct(op, bt, pc)
    torch.cuda.synchronize()
    lib.h2b_hara_phase_sync(0)
    for _ in range(a.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = peel_construct(op, bt, pc)
        torch.cuda.synchronize()
        t = time.perf_counter() - t0
        ph = (C.c_double * 16)()
        lib.h2b_hara_phase_ms(ph, 16)
        parts = ", ".join(f"{k} {ph[i]:.1f}" for i, k in enumerate(NAMES))
        print(f"build {t * 1e3:.1f} ms (op events {res.op_ms:.1f} ms): {parts}", flush=True)


if __name__ == "__main__":
    main()
