"""Where an NS inversion (cfg5 recipe) spends its time: HARA phase host times
(h2b_hara_phase_ms, no stream draining) summed over every Newton-Schulz iteration,
plus hgemv plan-build time. python tools/ns_phases.py [--surface 128]"""
import argparse
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2003_10173_b200 import PeelConfig  # noqa: E402
from paper_2003_10173_b200._lib import lib  # noqa: E402

NAMES = ["rng", "op_apply", "residual_hgemv", "absorb", "transposed_pass", "local_updates", "recompress",
         "dense_leaves", "orthogonalize", "truncation_bases", "projection"]

ap = argparse.ArgumentParser()
ap.add_argument("--surface", type=int, default=128)
a = ap.parse_args()
cfg = dict(bench.CONFIGS["cfg5"])
o, a0, X = bench.inversion_problem(a.surface, cfg)
pc = PeelConfig(eps=cfg["eps"], rng=1)
bench.inversion_step(a0, X, cfg, pc)   # warm-up
st0 = (C.c_ulonglong * 5)()
lib.h2b_jacobi_stats(st0)
lib.h2b_hara_phase_reset()
lib.h2b_plan_build_ms.restype = C.c_double
lib.h2b_plan_build_ms(1)
t0 = time.perf_counter()
t, res, au = bench.inversion_step(a0, X, cfg, pc)
wall = time.perf_counter() - t0
ph = (C.c_double * 16)()
lib.h2b_hara_phase_ms(ph, 16)
print(f"surface{a.surface}: wall {wall:.3f} s, steps {t}, iterations {len(res.trace.rows)}, "
      f"samples {res.trace.total_samples()}")
for i, nm in enumerate(NAMES):
    print(f"  {nm:18s} {ph[i] / 1e3:8.3f} s")
print(f"  hgemv plan builds  {lib.h2b_plan_build_ms(1) / 1e3:8.3f} s")
st1 = (C.c_ulonglong * 5)()
lib.h2b_jacobi_stats(st1)
sw, pr, cap, wsw, wpr = (st1[i] - st0[i] for i in range(5))
print(f"  jacobi: {pr} problems, {sw / max(pr, 1):.2f} sweeps on average, {cap} hit the sweep cap; "
      f"{wpr} with >= 64 columns: {wsw / max(wpr, 1):.2f} sweeps on average")
