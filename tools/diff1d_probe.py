"""Probe the device diffusion Hessian at cfg3 scale: setup time, per-apply
time at panel widths, and parity of a few columns against the CPU oracle."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2003_10173_b200 import Diffusion1D


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=262144)
    ap.add_argument("--steps", type=int, default=64)
    ap.add_argument("--b", type=int, nargs="+", default=[1, 16, 32, 64])
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--check", type=int, default=2)
    ap.add_argument("--tune", nargs="*", default=[], help="cpb:batch pairs to sweep (chunks per step CTA cap, columns per batch)")
    a = ap.parse_args()
    torch.cuda.init()
    t = time.perf_counter()
    d = Diffusion1D(n=a.n, steps=a.steps)
    torch.cuda.synchronize()
    print(f"setup {time.perf_counter() - t:.3f} s  nstate {d.nstate()}")
    from paper_2003_10173_b200._lib import lib
    combos = [tuple(int(v) for v in t.split(":")) for t in a.tune] or [(0, 0)]
    for cpb, batch in combos:
      if cpb:
        lib.h2b_diff1d_tune(cpb, batch)
        print(f"-- cpb<= {cpb}, batch {batch}")
      for b in a.b:
        x = torch.randn(b, a.n, dtype=torch.float64, device="cuda")
        y = torch.empty_like(x)
        d.hessvec_device(x.data_ptr(), y.data_ptr(), b)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            d.hessvec_device(x.data_ptr(), y.data_ptr(), b)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        print(f"b={b:3d}  {ms:9.3f} ms/apply  {ms / b:8.3f} ms/column")
    if a.check:
        from oracle import pyoracle as O
        ora = O.Diff1D(n=a.n, steps=a.steps)
        x = O.gaussian(11, a.n, a.check)
        t = time.perf_counter()
        yo = ora.hessvec(x, threads=a.check)
        tc = time.perf_counter() - t
        y = d.hessvec_at_target(x)
        r = np.linalg.norm(y - yo) / np.linalg.norm(yo)
        print(f"oracle {tc:.2f} s for {a.check} columns on {a.check} threads; rel diff {r:.3e}")


if __name__ == "__main__":
    main()
