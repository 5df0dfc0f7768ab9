import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
from paper_2003_10173_b200 import PeelConfig, ThresholdSchedule, h_newton_schulz, low_rank_update, recompress, scaled_identity_start
cfg = dict(bench.CONFIGS["cfg5"]); g = int(sys.argv[1]) if len(sys.argv) > 1 else 64
o, a0, X = bench.inversion_problem(g, cfg)
m = recompress(a0, 1e-12); m.add_diagonal(cfg["alpha"]); au = low_rank_update(recompress(m, 1e-8), X, X, 1e-8)
torch.cuda.synchronize()
t0 = time.perf_counter()
res = h_newton_schulz(au, scaled_identity_start(au), ThresholdSchedule(dynamic=True), cfg["eps"], PeelConfig(eps=cfg["eps"], rng=1), max_iter=int(sys.argv[2]) if len(sys.argv) > 2 else 64)
torch.cuda.synchronize()
print("NS s", time.perf_counter() - t0, len(res.trace.rows))
