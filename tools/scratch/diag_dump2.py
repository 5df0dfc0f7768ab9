import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from oracle import pyoracle as O
from paper_2003_10173_b200 import build_cluster_tree
pts = O.grid2d(32, 32); n = 1024
ct = build_cluster_tree(pts, 32)
inv = np.empty(n, np.int64); inv[ct.perm] = np.arange(n)
lv2 = [v for v in range(ct.num_nodes) if ct.level[v] == 2]
def owner(i):  # user index -> level-2 cluster
    ii = inv[i]
    for v in lv2:
        if ct.begin[v] <= ii < ct.end[v]: return v
g = np.fromfile("/tmp/pd_gpu_u2.bin").reshape(n, n, order="F")
o = np.fromfile("/tmp/pd_ora_u2.bin").reshape(n, n, order="F")
g1 = np.fromfile("/tmp/pd_gpu_r1.bin").reshape(n, n, order="F")
d = np.abs(g - o)
blk = {}
for a in lv2:
    ra = ct.perm[ct.begin[a]:ct.end[a]]
    for b in lv2:
        rb = ct.perm[ct.begin[b]:ct.end[b]]
        blk[(a, b)] = (np.linalg.norm(d[np.ix_(ra, rb)]), np.linalg.norm((g - g1)[np.ix_(ra, rb)]), np.linalg.norm((o - g1)[np.ix_(ra, rb)]))
for k, v in sorted(blk.items()): print(k, "diff %.3e  gpu-upd %.3e  ora-upd %.3e" % v)
print("level2 nodes", lv2, "children of 1:", ct.child0[1], ct.child1[1], "of 32:", ct.child0[32], ct.child1[32])
