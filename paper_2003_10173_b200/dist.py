"""Row-subtree sharded hgemv across GPUs: one process per GPU,
torch.distributed (NCCL over NVLink) for the single all-to-all exchange per
hgemv; every compute step runs in lib/libh2b200.so.

Rank r of P owns the subtree under the r-th node of level log2 P (its rows of
x and y); the top log2 P levels are replicated. The exchange carries the
x-hat of remote clusters that owned couplings / the replicated top upsweep read
and the x rows of remote near-field leaves (h2c.h, h2c_dist_*). It runs either
through torch.distributed (all_to_all_single) or, with transport="peer", as P2P
writes straight into the other GPUs' receive buffers with device-side signals
(h2c_dist_peer_*), so the exchange rides inside the begin / end kernels."""
import ctypes as C

import numpy as np

from ._lib import H, check, lib
from .h2 import col_major_geom


def partition_owner(bt, nranks):
    """Owning rank per cluster node (-1 = replicated top level); host only."""
    out = np.empty(bt.tree.num_nodes, np.int32)
    check(lib.h2c_partition_owner(bt._h, int(nranks), out.ctypes.data_as(C.c_void_p)))
    return out


def partition_exchange(bt, symmetric, up_ranks, nranks, src, dst, transpose=False):
    """Items rank dst receives from rank src: list of (arr, node, rows); host only."""
    ur = np.ascontiguousarray(up_ranks, np.int32)
    cnt = C.c_int64()
    check(lib.h2c_partition_exchange(bt._h, int(symmetric), int(transpose), ur.ctypes.data_as(C.c_void_p),
                                     int(nranks), int(src), int(dst), C.byref(cnt), None, None, None))
    arr = np.empty(cnt.value, np.int32)
    node = np.empty(cnt.value, np.int32)
    rows = np.empty(cnt.value, np.int64)
    if cnt.value:
        check(lib.h2c_partition_exchange(bt._h, int(symmetric), int(transpose), ur.ctypes.data_as(C.c_void_p),
                                         int(nranks), int(src), int(dst), C.byref(cnt),
                                         arr.ctypes.data_as(C.c_void_p), node.ctypes.data_as(C.c_void_p),
                                         rows.ctypes.data_as(C.c_void_p)))
    return list(zip(arr.tolist(), node.tolist(), rows.tolist()))


class DistPlan:
    """h2c_dist_plan: this rank's share of y = H x."""

    def __init__(self, m, nranks, rank, transpose=False):
        h = H()
        check(lib.h2c_dist_plan_create(m._h, int(transpose), int(nranks), int(rank), C.byref(h)))
        self._h = h
        self.matrix = m
        self.nranks, self.rank = int(nranks), int(rank)
        s = np.zeros(nranks, np.int64)
        r = np.zeros(nranks, np.int64)
        ob, orows = C.c_int64(), C.c_int64()
        check(lib.h2c_dist_plan_counts(h, s.ctypes.data_as(C.c_void_p), r.ctypes.data_as(C.c_void_p),
                                       C.byref(ob), C.byref(orows)))
        self.send_rows, self.recv_rows = s, r
        self.owned_begin, self.owned_rows = ob.value, orows.value

    def __del__(self):
        if getattr(self, "_h", None):
            lib.h2c_dist_plan_destroy(self._h)
            self._h = None

    def launches(self):
        v = C.c_int()
        check(lib.h2c_dist_plan_launches(self._h, C.byref(v)))
        return v.value

    def hgemv_nccl(self, comm, x, y, b, alpha=1.0, beta=0.0, stream=None, owned=False):
        """The whole sharded hgemv with the exchange on an ncclComm_t handle (an int / c_void_p
        from the process's NCCL), done inside the library (h2c_dist_hgemv_nccl)."""
        _, ldx = col_major_geom(x)
        _, ldy = col_major_geom(y)
        fn = lib.h2c_dist_hgemv_nccl_owned if owned else lib.h2c_dist_hgemv_nccl
        check(fn(self._h, comm, int(b), x.data_ptr(), ldx, y.data_ptr(), ldy, float(alpha), float(beta), stream))

    # ---- peer transport (h2c_dist_peer_*): P2P writes + signals, no collective call
    def peer_alloc(self, max_b):
        check(lib.h2c_dist_peer_alloc(self._h, int(max_b)))

    def peer_export(self):
        """(128 bytes of CUDA IPC handles, this rank's receive offsets in rows)."""
        hb = (C.c_char * 128)()
        off = np.zeros(self.nranks, np.int64)
        check(lib.h2c_dist_peer_export(self._h, C.cast(hb, C.c_void_p), off.ctypes.data_as(C.c_void_p)))
        return bytes(hb), off

    def peer_import(self, handles, offsets):
        """handles: every rank's export bytes (rank order); offsets: every rank's offsets."""
        hb = b"".join(handles)
        off = np.ascontiguousarray(np.stack(offsets), np.int64)
        check(lib.h2c_dist_peer_import(self._h, C.c_char_p(hb), off.ctypes.data_as(C.c_void_p)))

    @staticmethod
    def peer_link(plans):
        """Link the plans of every rank held by this process (ranks 0..P-1, tests)."""
        arr = (C.c_void_p * len(plans))(*[C.cast(p._h, C.c_void_p).value for p in plans])
        check(lib.h2c_dist_peer_link(arr, len(plans)))

    def begin(self, x, sendbuf, b, stream=None, owned=False):
        """owned: x holds only this rank's owned_rows rows, in cluster order.
        sendbuf None: peer transport (requires peer setup)."""
        _, ldx = col_major_geom(x)
        fn = lib.h2c_dist_hgemv_begin_owned if owned else lib.h2c_dist_hgemv_begin
        check(fn(self._h, int(b), x.data_ptr(), ldx, None if sendbuf is None else sendbuf.data_ptr(), stream))

    def local(self, b, stream=None):
        """Near-field products with this rank's own source rows (overlaps the exchange)."""
        check(lib.h2c_dist_hgemv_local(self._h, int(b), stream))

    def end(self, recvbuf, y, b, alpha=1.0, beta=0.0, stream=None, owned=False):
        """recvbuf None: peer transport (requires peer setup)."""
        _, ldy = col_major_geom(y)
        fn = lib.h2c_dist_hgemv_end_owned if owned else lib.h2c_dist_hgemv_end
        check(fn(self._h, int(b), None if recvbuf is None else recvbuf.data_ptr(), y.data_ptr(), ldy, float(alpha),
                 float(beta), stream))


class ShardedHgemv:
    """y = alpha H x + beta y for this rank's rows, exchange over torch.distributed.

    x, y: column-major (n x b, stride(0) == 1) float64 CUDA tensors holding the
    full user-ordered vectors; only owned rows of x are read and of y written.

    One hgemv: begin (gather, owned upsweep, pack) -> the all-to-all, issued
    asynchronously -> local near field on the compute stream while it is in
    flight -> wait -> end (unpack, couplings, downsweep, remaining near field,
    leaf expansion). NCCL groups exchange device buffers (the collective runs
    on NCCL's stream, concurrent with the local near field); other backends
    (gloo) stage the buffers through host memory."""

    def __init__(self, m, group=None, transpose=False, transport="collective", max_b=64):
        """transport "collective": the all-to-all through torch.distributed (NCCL on
        device buffers, host-staged for gloo); "peer": P2P writes into the other GPUs'
        receive buffers with device-side signals (CUDA IPC handles exchanged once
        with an allgather over `group`; every GPU must be peer-accessible)."""
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.plan = DistPlan(m, world, rank, transpose)
        self.device_collective = dist.is_initialized() and dist.get_backend(group) == "nccl"
        self._bufs = {}
        if transport not in ("collective", "peer"):
            raise ValueError("transport must be 'collective' or 'peer'")
        self.peer = transport == "peer" and world > 1
        self.max_b = int(max_b)
        if self.peer:
            self.plan.peer_alloc(self.max_b)
            mine = self.plan.peer_export()
            allv = [None] * world
            dist.all_gather_object(allv, mine, group=group)
            self.plan.peer_import([a[0] for a in allv], [a[1] for a in allv])

    def _buffers(self, b, device):
        import torch
        key = (b, str(device))
        if key not in self._bufs:
            self._bufs[key] = (torch.empty(max(1, int(self.plan.send_rows.sum()) * b), dtype=torch.float64, device=device),
                               torch.empty(max(1, int(self.plan.recv_rows.sum()) * b), dtype=torch.float64, device=device))
        return self._bufs[key]

    def __call__(self, x, y, alpha=1.0, beta=0.0, owned=False):
        """owned=False: x, y are the full user-ordered vectors (n rows); owned=True:
        only this rank's plan.owned_rows rows, in cluster order."""
        import torch
        b = x.shape[1] if x.dim() == 2 else 1
        s = torch.cuda.current_stream(x.device).cuda_stream
        if self.peer:   # the exchange is device-side: no host call between begin and end
            if b > self.max_b:
                raise ValueError(f"peer transport: b={b} exceeds max_b={self.max_b}")
            self.plan.begin(x, None, b, s, owned)
            self.plan.local(b, s)
            self.plan.end(None, y, b, alpha, beta, s, owned)
            return
        send, recv = self._buffers(b, x.device)
        self.plan.begin(x, send, b, s, owned)
        if self.plan.nranks > 1:
            ns, nr = int(self.plan.send_rows.sum()) * b, int(self.plan.recv_rows.sum()) * b
            osz = [int(v) * b for v in self.plan.recv_rows]
            isz = [int(v) * b for v in self.plan.send_rows]
            if self.device_collective:
                work = self.dist.all_to_all_single(recv[:nr], send[:ns], output_split_sizes=osz,
                                                   input_split_sizes=isz, group=self.group, async_op=True)
                self.plan.local(b, s)   # on the compute stream, beside NCCL's
                work.wait()             # the compute stream waits for the exchange
            else:
                self.plan.local(b, s)
                hs = send[:ns].cpu()    # synchronises the compute stream
                hr = torch.empty(nr, dtype=torch.float64)
                self.dist.all_to_all_single(hr, hs, output_split_sizes=osz, input_split_sizes=isz, group=self.group)
                recv[:nr].copy_(hr)
        self.plan.end(recv, y, b, alpha, beta, s, owned)
