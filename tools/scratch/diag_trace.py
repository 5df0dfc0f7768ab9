import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from oracle import pyoracle as O
from paper_2003_10173_b200 import *
pts = O.grid2d(32, 32); n = 1024
r = np.sqrt(((pts[:, None, :] - pts[None, :, :]) ** 2).sum(-1))
a = np.exp(-r / 0.2) + 0.5 * np.eye(n)
ct = build_cluster_tree(pts, 32); bt = build_block_tree(ct, ct, 1.0)
which = sys.argv[1]
if which == "gpu":
    res = peel_construct(DenseOperator(a, True), bt, PeelConfig(eps=1e-5, norm_scale=3.0))
else:
    O.peel_dense(O.Tree(pts, 32), a, True, eps=1e-5, norm_scale=3.0)
