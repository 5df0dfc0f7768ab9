import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from oracle import pyoracle as O, pyref as R
from paper_2003_10173_b200 import *
for case in ("1d", "2d"):
    pts, leaf, weak = (O.grid1d(200, -1, 1), 12, True) if case == "1d" else (O.grid2d(24, 24), 16, False)
    for sym in (True, False):
        ref = O.Tree(pts, leaf, 1.0, weak); rr_ = R.Tree(pts, leaf, 1.0, weak)
        ora = O.H2.random(ref, sym, 12, 21); orr = R.H2.random(rr_, sym, 12, 21)
        ct = build_cluster_tree(pts, leaf); bt = build_block_tree(ct, ct, 1.0, Admissibility.weak if weak else Admissibility.strong)
        rr, cr = ora.ranks()
        m = H2Matrix.from_packed(bt, sym, rr, cr, ora.export())
        go = orthogonalize(m).ranks()[0]; oo = ora.orthogonalize().ranks()[0]
        print(case, sym, "orth ranks equal", np.array_equal(go, oo))
        for eps in (0.3, 0.1, 1e-2, 1e-3):
            g = recompress(m, eps).ranks()[0]; o = ora.recompress(eps).ranks()[0]; r = orr.recompress(eps).ranks()[0]
            d = np.nonzero(g != o)[0]
            print(case, sym, eps, "gpu==ora", np.array_equal(g, o), "ora==ref", np.array_equal(o, r), "ndiff", len(d), d[:8], g[d[:8]], o[d[:8]])
