import sys, os, time, ctypes as C
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
from paper_2003_10173_b200._lib import lib
cfg = dict(bench.CONFIGS["cfg5"]); g = int(sys.argv[1]) if len(sys.argv) > 1 else 128
from paper_2003_10173_b200 import PeelConfig
o, a0, X = bench.inversion_problem(g, cfg)
pc = PeelConfig(eps=cfg["eps"], rng=1)
bench.inversion_step(a0, X, cfg, pc)
lib.h2b_hara_phase_sync(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
ph = (C.c_double * 16)(); lib.h2b_hara_phase_reset(); lib.h2b_hara_phase_ms(ph, 16)
lib.h2b_plan_build_ms.restype = C.c_double; lib.h2b_plan_build_ms.argtypes = [C.c_int]; lib.h2b_plan_build_ms(1)
base = list(ph)
t0 = time.perf_counter()
t, res, au = bench.inversion_step(a0, X, cfg, pc)
tot = time.perf_counter() - t0
lib.h2b_hara_phase_ms(ph, 16)
names = ["rng", "op_apply", "residual_hgemv", "absorb", "transposed_pass", "local_updates", "recompress", "dense_leaves", "orthogonalize_all", "truncation_bases", "projection"]
print("total", round(tot, 3), t, "iters", len(res.trace.rows), "samples", res.trace.total_samples())
print({n: round((ph[i] - base[i]) / 1e3, 3) for i, n in enumerate(names)}, "plan builds s", round(lib.h2b_plan_build_ms(0) / 1e3, 3))
