import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2003_10173_b200 import *
import bench
pts = bench.grid_points((262144,))
ct = build_cluster_tree(pts, 32); bt = build_block_tree(ct, ct, 1.0, Admissibility.weak)
m = H2Matrix.kernel(bt, pts, "gaussian", 0.05, 16)
g = orthogonalize(m)
torch.cuda.synchronize()
for i in range(3):
    t = time.perf_counter(); r = recompress(g, 1e-7); torch.cuda.synchronize(); print("recompress ms", (time.perf_counter() - t) * 1e3)
from paper_2003_10173_b200._lib import lib
for knob in (0, 1, 0, 1):
    lib.h2b_la_tune(0, knob)
    t = time.perf_counter(); r = recompress(g, 1e-7); torch.cuda.synchronize()
    print("jacobi_warp", knob, "recompress ms", round((time.perf_counter() - t) * 1e3, 2), "ranks", r.rank_profile().tolist())
