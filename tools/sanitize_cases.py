"""Small runs of the paths compute-sanitizer should see (one tool per call):
the few-vector b<=2 path (dense pass overlapped with the sweep chain, bulk-async
ring variant, slot sums), the b=32 path with graph replay, the split stage 5,
the sharded begin/local/end sequence, and one HARA build.

  compute-sanitizer --tool memcheck  python tools/sanitize_cases.py
  compute-sanitizer --tool racecheck python tools/sanitize_cases.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from oracle import pyoracle as O
from paper_2003_10173_b200 import (Admissibility, DenseOperator, H2Matrix, PeelConfig, build_block_tree,
                                   build_cluster_tree, peel_construct)
from paper_2003_10173_b200._lib import lib
from paper_2003_10173_b200.dist import DistPlan


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


pts = O.grid2d(256, 256)   # 1024 leaves: enough dense blocks for the bulk-async ring variant
ct = build_cluster_tree(pts, 64)
bt = build_block_tree(ct, ct, 1.0)
m = H2Matrix.kernel(bt, pts, "gaussian", 0.1, 16)
n = pts.shape[0]
ref = O.H2.from_packed(O.Tree(pts, 64), True, m.ranks()[0], None, m.download())
for b in (1, 2, 32):
    x = O.gaussian(b, n, b)
    xt = torch.from_numpy(x.T.copy()).cuda().t()
    for rep in range(3):   # eager, graph capture, graph replay
        yt = torch.zeros(b, n, dtype=torch.float64, device="cuda").t()
        m.hgemv(xt, yt)
    torch.cuda.synchronize()
    print("hgemv b", b, "rel err", rel(yt.cpu().numpy(), ref.matvec(x)), flush=True)
lib.h2b_tune(9, 1)   # split stage 5 on one GPU
x = O.gaussian(7, n, 16)
xt = torch.from_numpy(x.T.copy()).cuda().t()
yt = torch.zeros(16, n, dtype=torch.float64, device="cuda").t()
m.hgemv(xt, yt)
torch.cuda.synchronize()
lib.h2b_tune(9, 0)
print("split rel err", rel(yt.cpu().numpy(), ref.matvec(x)), flush=True)
plans = [DistPlan(m, 2, r) for r in range(2)]
sends = [torch.zeros(max(1, int(p.send_rows.sum()) * 16), dtype=torch.float64, device="cuda") for p in plans]
for p, sb in zip(plans, sends):
    p.begin(xt, sb, 16)
    p.local(16)
yt.zero_()
for r, p in enumerate(plans):
    recv = torch.cat([sends[q][int(pq.send_rows[:r].sum()) * 16:int(pq.send_rows[:r + 1].sum()) * 16]
                      for q, pq in enumerate(plans)])
    p.end(recv if recv.numel() else torch.zeros(1, dtype=torch.float64, device="cuda"), yt, 16)
torch.cuda.synchronize()
print("sharded rel err", rel(yt.cpu().numpy(), ref.matvec(x)), flush=True)
p1 = O.grid1d(512, -1, 1)
c1 = build_cluster_tree(p1, 16)
b1 = build_block_tree(c1, c1, 1.0, Admissibility.weak)
a = np.exp(-np.abs(p1 - p1.T) / 0.3) + 0.5 * np.eye(512)
res = peel_construct(DenseOperator(a, True), b1, PeelConfig(eps=1e-6))
torch.cuda.synchronize()
print("peel samples", res.stats.total, flush=True)
