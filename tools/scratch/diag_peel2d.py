import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from oracle import pyoracle as O
from paper_2003_10173_b200 import *
pts = O.grid2d(32, 32); n = 1024
r = np.sqrt(((pts[:, None, :] - pts[None, :, :]) ** 2).sum(-1))
a = np.exp(-r / 0.2) + 0.5 * np.eye(n)
ct = build_cluster_tree(pts, 32); bt = build_block_tree(ct, ct, 1.0)
op = DenseOperator(a, True)
print("pnorm gpu", pnorm_estimate(op, 2), "cpu", O.pnorm2_dense(a, True))
for eps in (1e-5, 1e-6, 1e-4, 3e-5):
    for ns in (0.0, 3.0):
        res = peel_construct(DenseOperator(a, True), bt, PeelConfig(eps=eps, norm_scale=ns))
        ho, so = O.peel_dense(O.Tree(pts, 32), a, True, eps=eps, norm_scale=ns)
        gl = [lv.samples for lv in res.stats.levels]
        gr = [lv.max_rank for lv in res.stats.levels]
        rg = res.matrix.ranks()[0]; ro = ho.ranks()[0]
        d = np.nonzero(rg != ro)[0]
        print(eps, ns, gl == so["level_samples"], gl, so["level_samples"], gr, so["level_max_rank"], "rankdiff nodes", d[:10], rg[d[:10]], ro[d[:10]])
