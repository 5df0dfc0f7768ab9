"""Sharded (row-subtree) hgemv host logic on CPU with torch.distributed/gloo,
world sizes 2 and 4.

The partition (owner per node) and the exchange lists come from the product
library's host code (h2c_partition_owner / h2c_partition_exchange — the same
functions the device plans use); each gloo rank then runs the sharded
algorithm in numpy on the oracle's payload (test infrastructure) and the
assembled y must equal the oracle's unsharded hgemv."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class NumpyH2:
    """Per-node view of an oracle export (layout of include/h2c.h)."""

    def __init__(self, ref, ranks, parts, symmetric):
        self.t, self.k, self.sym = ref, np.asarray(ranks), symmetric
        nn = ref.num_nodes
        leaves = [v for v in range(nn) if ref.child0[v] < 0]
        size = lambda v: int(ref.end[v] - ref.begin[v])
        self.U, self.E, self.S, self.D = {}, {}, {}, {}
        o = 0
        for v in leaves:
            m, k = size(v), int(self.k[v])
            self.U[v] = parts["U"][o:o + m * k].reshape((m, k), order="F")
            o += m * k
        o = 0
        for v in range(nn):
            p = ref.parent[v]
            if p < 0:
                continue
            a, b = int(self.k[v]), int(self.k[p])
            self.E[v] = parts["E"][o:o + a * b].reshape((a, b), order="F")
            o += a * b
        stores = lambda b: (not symmetric) or ref.brow[b] <= ref.bcol[b]
        o = 0
        for b in ref.adm:
            if not stores(b):
                continue
            a, c = int(self.k[ref.brow[b]]), int(self.k[ref.bcol[b]])
            self.S[b] = parts["S"][o:o + a * c].reshape((a, c), order="F")
            o += a * c
        o = 0
        for b in ref.dense:
            if not stores(b):
                continue
            a, c = size(ref.brow[b]), size(ref.bcol[b])
            self.D[b] = parts["D"][o:o + a * c].reshape((a, c), order="F")
            o += a * c
        self.leaves = leaves

    def orient(self, blocks):
        for b, M in blocks.items():
            r, c = int(self.t.brow[b]), int(self.t.bcol[b])
            yield r, c, M
            if self.sym and r != c:
                yield c, r, M.T


def _sharded_rank(rank, world, port, case, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import sys
    sys.path.insert(0, ROOT)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import pyoracle as O
        from paper_2003_10173_b200 import Admissibility, build_block_tree, build_cluster_tree
        from paper_2003_10173_b200.dist import partition_exchange, partition_owner
        pts, leaf, weak = case
        ref = O.Tree(pts, leaf, 1.0, weak)
        ora = O.H2.random(ref, True, 6, 17)
        rr, _ = ora.ranks()
        h = NumpyH2(ref, rr, ora.export(), True)
        ct = build_cluster_tree(pts, leaf)
        bt = build_block_tree(ct, ct, 1.0, Admissibility.weak if weak else Admissibility.strong)
        owner = partition_owner(bt, world)
        n, b = pts.shape[0], 3
        x = O.gaussian(5, n, b)
        xi = x[ref.perm]
        t = ref
        local = lambda v: owner[v] == rank or owner[v] < 0
        lp = int(np.log2(world))
        xhat = {}
        # phase A: owned leaves + owned upsweep
        for lvl in range(t.depth, lp - 1, -1):
            for v in range(t.num_nodes):
                if t.level[v] != lvl or owner[v] != rank:
                    continue
                if t.child0[v] < 0:
                    xhat[v] = h.U[v].T @ xi[t.begin[v]:t.end[v]]
                else:
                    xhat[v] = sum(h.E[c].T @ xhat[c] for c in (t.child0[v], t.child1[v]))
        # exchange exactly the items the library lists, in its order
        out = {}
        for dst in range(world):
            items = partition_exchange(bt, True, rr, world, rank, dst)
            out[dst] = [xi[t.begin[v]:t.end[v]] if a == 0 else xhat[v] for a, v, _ in items]
            for (a, v, rows), blk in zip(items, out[dst]):
                assert blk.shape[0] == rows
        gathered = [None] * world
        dist.all_gather_object(gathered, out)
        for src in range(world):
            items = partition_exchange(bt, True, rr, world, src, rank)
            for (a, v, _), blk in zip(items, gathered[src][rank]):
                if a == 0:
                    xi[t.begin[v]:t.end[v]] = blk
                else:
                    xhat[v] = blk
        # phase B: replicated top upsweep, couplings, downsweep, owned leaves
        for lvl in range(lp - 1, -1, -1):
            for v in range(t.num_nodes):
                if t.level[v] == lvl:
                    xhat[v] = sum(h.E[c].T @ xhat[c] for c in (t.child0[v], t.child1[v]))
        yhat = {v: np.zeros((int(h.k[v]), b)) for v in range(t.num_nodes) if local(v)}
        for r, c, M in h.orient(h.S):
            if local(r):
                yhat[r] += M @ xhat[c]
        for lvl in range(t.depth + 1):
            for v in range(t.num_nodes):
                if t.level[v] != lvl or not local(v) or t.child0[v] < 0:
                    continue
                for c in (t.child0[v], t.child1[v]):
                    if local(c):
                        yhat[c] += h.E[c] @ yhat[v]
        yi = {}
        for v in h.leaves:
            if owner[v] != rank:
                continue
            yi[v] = h.U[v] @ yhat[v]
        for r, c, M in h.orient(h.D):
            if owner[r] == rank:
                yi[r] = yi[r] + M @ xi[t.begin[c]:t.end[c]]
        parts = [None] * world
        dist.all_gather_object(parts, yi)
        if rank == 0:
            y_int = np.zeros((n, b))
            for p in parts:
                for v, blk in p.items():
                    y_int[t.begin[v]:t.end[v]] = blk
            y = np.empty_like(y_int)
            y[t.perm] = y_int
            ref_y = ora.matvec(x)
            q.put(float(np.linalg.norm(y - ref_y) / np.linalg.norm(ref_y)))
    except Exception as e:  # report into the parent
        if rank == 0:
            q.put(repr(e))
        raise
    finally:
        dist.destroy_process_group()


def _cases():
    from oracle import pyoracle as O
    return {"2d-strong": (O.grid2d(32, 32), 16, False), "1d-weak": (O.grid1d(512, -1, 1), 16, True)}


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("case", ["2d-strong", "1d-weak"])
def test_sharded_hgemv_gloo(world, case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_rank, args=(r, world, port, _cases()[case], q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    assert not isinstance(res, str), res
    assert res <= 1e-13, res


def test_partition_owner_covers_tree():
    from oracle import pyoracle as O
    from paper_2003_10173_b200 import build_block_tree, build_cluster_tree
    from paper_2003_10173_b200.dist import partition_owner
    pts = O.grid2d(64, 64)
    ct = build_cluster_tree(pts, 32)
    bt = build_block_tree(ct, ct, 1.0)
    for world in (1, 2, 4, 8):
        own = partition_owner(bt, world)
        lp = int(np.log2(world))
        assert np.all(own[ct.level < lp] == -1)
        assert np.all(own[ct.level >= lp] >= 0)
        # owned row ranges tile the points evenly (median splits)
        sizes = [int((ct.end[ct.leaves][own[ct.leaves] == r] - ct.begin[ct.leaves][own[ct.leaves] == r]).sum())
                 for r in range(world)]
        assert sum(sizes) == ct.n and max(sizes) - min(sizes) <= 1 * world
    with pytest.raises(ValueError):
        partition_owner(bt, 3)
