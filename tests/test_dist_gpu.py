"""Sharded hgemv on the B200: P ranks simulated on one GPU (each with its own
plan, workspace and buffers; the all-to-all is done by device copies in rank
order, exactly the layout torch.distributed.all_to_all_single uses), and a real
two-process run of ShardedHgemv over a gloo group (host-staged exchange; both
processes on cuda:0, which is safe because no kernel waits on the other rank).
The sharded plan splits the near field into local-source partial sums (run
while the exchange is in flight) and remote-source ones, so its sum order
differs from the single-GPU plan: <= 1e-13 relative, every P."""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2003_10173_b200 import Admissibility, H2Matrix, build_block_tree, build_cluster_tree
from paper_2003_10173_b200.dist import DistPlan

pytestmark = pytest.mark.gpu


def close(y, y_ref, P):
    # sharded plans always split the near field (local-source partial sums run while
    # the exchange is in flight), so the sum order differs from the single-GPU plan
    return float((y - y_ref).abs().max()) <= 1e-13 * float(y_ref.abs().max())


def simulate(m, P, x, y, b, transpose=False, alpha=1.0, beta=0.0, local=False):
    import torch
    plans = [DistPlan(m, P, r, transpose) for r in range(P)]
    sends = [torch.zeros(max(1, int(p.send_rows.sum()) * b), dtype=torch.float64, device=x.device) for p in plans]
    for p, s in zip(plans, sends):
        p.begin(x, s, b)
        if local:
            p.local(b)
    for r, p in enumerate(plans):
        segs = []
        for q, pq in enumerate(plans):
            off = int(pq.send_rows[:r].sum()) * b
            assert int(pq.send_rows[r]) == int(p.recv_rows[q])
            segs.append(sends[q][off:off + int(pq.send_rows[r]) * b])
        recv = torch.cat(segs) if segs else torch.zeros(1, dtype=torch.float64, device=x.device)
        if recv.numel() == 0:
            recv = torch.zeros(1, dtype=torch.float64, device=x.device)
        p.end(recv, y, b, alpha, beta)
    torch.cuda.synchronize()
    return plans


CASES = {
    "2d-strong-kernel": (lambda: O.grid2d(64, 64), 32, False),
    "1d-weak-random": (lambda: O.grid1d(2048, -1, 1), 32, True),
    "3d-strong-random": (lambda: O.grid3d(16, 16, 16), 32, False),
}


@pytest.mark.parametrize("P", [1, 2, 4, 8])
@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("sym", [True, False])
def test_sharded_equals_unsharded(cuda, P, case, sym):
    import torch
    mk, leaf, weak = CASES[case]
    pts = mk()
    ct = build_cluster_tree(pts, leaf)
    bt = build_block_tree(ct, ct, 1.0, Admissibility.weak if weak else Admissibility.strong)
    if case.endswith("kernel") and sym:
        m = H2Matrix.kernel(bt, pts, "gaussian", 0.1, 16)
    else:
        ref = O.Tree(pts, leaf, 1.0, weak)
        ora = O.H2.random(ref, sym, 12, 8)
        rr, cr = ora.ranks()
        m = H2Matrix.from_packed(bt, sym, rr, cr, ora.export())
    n, b = pts.shape[0], 32
    x = torch.randn(b, n, dtype=torch.float64, device=cuda).t()
    for transpose in ((False, True) if not sym else (False,)):
        y_ref = torch.zeros(b, n, dtype=torch.float64, device=cuda).t()
        m.hgemv(x, y_ref, transpose=transpose)
        y = torch.full((b, n), 7.0, dtype=torch.float64, device=cuda).t()
        plans = simulate(m, P, x, y, b, transpose, local=(P % 2 == 0))
        assert sum(p.owned_rows for p in plans) == n
        assert close(y, y_ref, P), float((y - y_ref).abs().max())


def test_sharded_exchange_volume_2d(cuda):
    # halo traffic is a small fraction of the matrix at P = 8
    pts = O.grid2d(256, 256)
    ct = build_cluster_tree(pts, 64)
    bt = build_block_tree(ct, ct, 1.0)
    m = H2Matrix.kernel(bt, pts, "gaussian", 0.1, 32)
    plans = [DistPlan(m, 8, r) for r in range(8)]
    recv = max(int(p.recv_rows.sum()) for p in plans)
    owned = pts.shape[0] // 8
    # measured 17,920 rows per vector column at this size (x-hat + x halo)
    assert recv <= 2.5 * owned, (recv, owned)


@pytest.mark.parametrize("P", [2, 4, 8])
def test_sharded_payload_equals_unsharded(cuda, P):
    # each rank generates only its shard's payload; the assembled y is bitwise the full hgemv
    import torch
    pts = O.grid2d(96, 96)
    ct = build_cluster_tree(pts, 32)
    bt = build_block_tree(ct, ct, 1.0)
    full = H2Matrix.kernel(bt, pts, "gaussian", 0.1, 16)
    n, b = pts.shape[0], 32
    x = torch.randn(b, n, dtype=torch.float64, device=cuda).t()
    y_ref = torch.zeros(b, n, dtype=torch.float64, device=cuda).t()
    full.hgemv(x, y_ref)
    shards = [H2Matrix.kernel(bt, pts, "gaussian", 0.1, 16, shard=(P, r)) for r in range(P)]
    plans = [DistPlan(shards[r], P, r) for r in range(P)]
    sends = [torch.zeros(max(1, int(p.send_rows.sum()) * b), dtype=torch.float64, device=cuda) for p in plans]
    for p, s in zip(plans, sends):
        p.begin(x, s, b)
    y = torch.full((b, n), 3.0, dtype=torch.float64, device=cuda).t()
    for r, p in enumerate(plans):
        segs = [sends[q][int(pq.send_rows[:r].sum()) * b:int(pq.send_rows[:r + 1].sum()) * b]
                for q, pq in enumerate(plans)]
        recv = torch.cat(segs)
        if recv.numel() == 0:
            recv = torch.zeros(1, dtype=torch.float64, device=cuda)
        p.end(recv, y, b)
    torch.cuda.synchronize()
    assert close(y, y_ref, P)
    fsz = sum(full.packed_sizes())
    ssz = [sum(s.packed_sizes()) for s in shards]
    assert max(ssz) < 0.8 * fsz and sum(ssz) < 1.6 * fsz   # payload is actually sharded
    with pytest.raises(ValueError):
        shards[0].hgemv(x, y)


@pytest.mark.parametrize("P", [1, 2, 4])
def test_sharded_owned_rows_layout(cuda, P):
    """begin_owned / end_owned: each rank passes only its owned rows, in cluster order."""
    import torch
    pts = O.grid2d(64, 64)
    ct = build_cluster_tree(pts, 32)
    bt = build_block_tree(ct, ct, 1.0)
    m = H2Matrix.kernel(bt, pts, "gaussian", 0.1, 16)
    n, b = pts.shape[0], 8
    x = torch.randn(b, n, dtype=torch.float64, device=cuda).t()
    y_ref = torch.zeros(b, n, dtype=torch.float64, device=cuda).t()
    m.hgemv(x, y_ref, ordering=1)          # internal (cluster) ordering on both sides
    plans = [DistPlan(m, P, r) for r in range(P)]
    sends = [torch.zeros(max(1, int(p.send_rows.sum()) * b), dtype=torch.float64, device=cuda) for p in plans]
    for p, sb in zip(plans, sends):
        xo = x[p.owned_begin:p.owned_begin + p.owned_rows].contiguous().t().contiguous().t()
        p.begin(xo, sb, b, owned=True)
    y = torch.zeros(b, n, dtype=torch.float64, device=cuda).t()
    for r, p in enumerate(plans):
        segs = [sends[q][int(pq.send_rows[:r].sum()) * b:int(pq.send_rows[:r + 1].sum()) * b]
                for q, pq in enumerate(plans)]
        recv = torch.cat(segs)
        if recv.numel() == 0:
            recv = torch.zeros(1, dtype=torch.float64, device=cuda)
        yo = torch.full((b, p.owned_rows), 5.0, dtype=torch.float64, device=cuda).t()
        p.end(recv, yo, b, owned=True)
        y[p.owned_begin:p.owned_begin + p.owned_rows] = yo
    torch.cuda.synchronize()
    assert close(y, y_ref, P)


def _two_rank_worker(rank, world, port, sym, q):
    import os
    import sys
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import pyoracle as O
        from paper_2003_10173_b200 import Admissibility, H2Matrix, build_block_tree, build_cluster_tree
        from paper_2003_10173_b200.dist import ShardedHgemv
        torch.cuda.set_device(0)
        pts = O.grid2d(48, 48)
        ref = O.Tree(pts, 24, 1.0, False)
        ora = O.H2.random(ref, sym, 10, 19)
        ct = build_cluster_tree(pts, 24)
        bt = build_block_tree(ct, ct, 1.0, Admissibility.strong)
        rr, cr = ora.ranks()
        m = H2Matrix.from_packed(bt, sym, rr, cr, ora.export())
        n, b = pts.shape[0], 6
        xh = O.gaussian(3, n, b)
        x = torch.from_numpy(xh.T.copy()).cuda().t()
        y = torch.zeros(b, n, dtype=torch.float64, device="cuda").t()
        sh = ShardedHgemv(m)             # the product's multi-process path, gloo group
        assert not sh.device_collective
        sh(x, y)
        sh(x, y, alpha=2.0, beta=-1.0)   # y = 2 H x - H x = H x again
        torch.cuda.synchronize()
        p = sh.plan
        own = torch.zeros(n, dtype=torch.float64)
        perm = ct.perm[p.owned_begin:p.owned_begin + p.owned_rows]
        part = y.cpu().numpy()[perm]
        parts = [None] * world
        dist.all_gather_object(parts, (perm, part))
        if rank == 0:
            yy = np.zeros((n, b))
            for pr, blk in parts:
                yy[pr] = blk
            yr = ora.matvec(xh)
            q.put(float(np.linalg.norm(yy - yr) / np.linalg.norm(yr)))
    except Exception as e:
        q.put(repr(e))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("sym", [True, False])
def test_sharded_hgemv_two_processes_gloo(cuda, sym):
    """ShardedHgemv.__call__ in two real processes (world 2, gloo, host-staged
    all-to-all) against the oracle: the multi-process path end to end."""
    import multiprocessing as mp
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_two_rank_worker, args=(r, 2, port, sym, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = q.get(timeout=240)
    for pr in procs:
        pr.join(timeout=120)
    assert isinstance(res, float), res
    assert res <= 1e-12


@pytest.mark.parametrize("P", [2, 4])
@pytest.mark.parametrize("case", list(CASES))
def test_peer_transport_equals_collective(cuda, P, case):
    """Peer transport (h2c_dist_peer_*): begin writes every send item straight into
    its destination plan's receive buffer and signals it; end waits for the signals,
    unpacks and acknowledges. The P plans live in this process on one GPU and are
    linked directly; all begins are enqueued before any end, so no kernel ever waits
    on work that has not already run. Three calls exercise the epoch counters and the
    acknowledgements; the result is bitwise the collective path's."""
    import torch
    mk, leaf, weak = CASES[case]
    pts = mk()
    ct = build_cluster_tree(pts, leaf)
    bt = build_block_tree(ct, ct, 1.0, Admissibility.weak if weak else Admissibility.strong)
    ref = O.Tree(pts, leaf, 1.0, weak)
    ora = O.H2.random(ref, False, 12, 8)
    rr, cr = ora.ranks()
    m = H2Matrix.from_packed(bt, False, rr, cr, ora.export())
    n, b = pts.shape[0], 5
    plans = [DistPlan(m, P, r) for r in range(P)]
    for p in plans:
        p.peer_alloc(8)
    DistPlan.peer_link(plans)
    for call in range(3):
        xc = torch.randn(b, n, dtype=torch.float64, device=cuda).t()
        y_coll = torch.zeros(b, n, dtype=torch.float64, device=cuda).t()
        simulate(m, P, xc, y_coll, b, local=True)
        y = torch.full((b, n), 3.0, dtype=torch.float64, device=cuda).t()
        for p in plans:
            p.begin(xc, None, b)
            p.local(b)
        for p in plans:
            p.end(None, y, b)
        torch.cuda.synchronize()
        assert torch.equal(y, y_coll), float((y - y_coll).abs().max())


def test_peer_transport_needs_setup(cuda):
    import torch
    pts = O.grid2d(32, 32)
    ct = build_cluster_tree(pts, 32)
    bt = build_block_tree(ct, ct, 1.0)
    m = H2Matrix.kernel(bt, pts, "gaussian", 0.1, 8)
    p = DistPlan(m, 2, 0)
    x = torch.randn(2, pts.shape[0], dtype=torch.float64, device=cuda).t()
    with pytest.raises(NotImplementedError):   # std::logic_error: no buffer and no peer transport
        p.begin(x, None, 2)


def test_nccl_entry_single_rank(cuda):
    """h2c_dist_hgemv_nccl on a one-rank NCCL communicator (ncclCommInitAll from the NCCL the
    process already loaded): the library resolves NCCL at run time, packs, exchanges nothing and
    matches the single-GPU hgemv. (More ranks need more GPUs than this environment has.)"""
    import ctypes as C
    import torch
    torch.zeros(1, device=cuda)
    import torch.cuda.nccl  # noqa: F401  loads torch's libnccl.so.2
    try:
        nccl = C.CDLL("libnccl.so.2", mode=C.RTLD_GLOBAL)
    except OSError:
        pytest.skip("no libnccl.so.2 in the process")
    comm = C.c_void_p()
    devs = (C.c_int * 1)(torch.cuda.current_device())
    assert nccl.ncclCommInitAll(C.byref(comm), 1, devs) == 0
    pts = O.grid2d(64, 64)
    ct = build_cluster_tree(pts, 32)
    bt = build_block_tree(ct, ct, 1.0)
    m = H2Matrix.kernel(bt, pts, "gaussian", 0.1, 12)
    n, b = pts.shape[0], 7
    x = torch.randn(b, n, dtype=torch.float64, device=cuda).t()
    y_ref = torch.zeros(b, n, dtype=torch.float64, device=cuda).t()
    m.hgemv(x, y_ref)
    p = DistPlan(m, 1, 0)
    y = torch.zeros(b, n, dtype=torch.float64, device=cuda).t()
    p.hgemv_nccl(comm, x, y, b)
    torch.cuda.synchronize()
    nccl.ncclCommDestroy(comm)
    assert close(y, y_ref, 1)
