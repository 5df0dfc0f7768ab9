import sys, os, subprocess
import numpy as np
n = 1024
for L in range(1, 6):
    for tag in ("u", "r"):
        g = np.fromfile(f"/tmp/pd_gpu_{tag}{L}.bin").reshape(n, n)
        o = np.fromfile(f"/tmp/pd_ora_{tag}{L}.bin").reshape(n, n)
        print(L, tag, "||g-o||/||o||", np.linalg.norm(g - o) / np.linalg.norm(o), "max", np.abs(g - o).max())
