#!/usr/bin/env python
"""hgemv benchmark (BASELINE.json metric: hgemv GFLOP/s + GB/s, N=2^20, 32
vectors, fp64; configs[1] = 2D Gaussian-kernel H^2, leaf 64, rank 32).

One step = one hgemv y = H x of the whole synthetic H^2 matrix over one batch
of b vectors (x resident in HBM). value = algorithmic GFLOP/s of the whole job
(max-over-ranks device time). Also reported: GB/s, the roofline of the
dominant kernel (leaf expansion + dense near-field, measured live with CUDA
events), the end-to-end host-buffer path (H2D x, hgemv, D2H y), and the CPU
oracle (port of the reference) timed on a bounded sample on the host cores.

  python bench.py [--gpus N --steps K --warmup W] [--config cfg2|cfg2b1|cfg1|cfg4] [--impl reference]
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
FLUSH_BYTES = 256 << 20   # > the B200's 126 MB L2
sys.path.insert(0, ROOT)

CONFIGS = {
    # BASELINE.json configs[1] (the metric's config)
    "cfg2": dict(workload="2D Gaussian-kernel H2 hgemv, N=2^20 (1024^2 grid on [0,1]^2), leaf 64, eta=1 strong, "
                          "rank 32, 32 vectors, fp64, symmetric canonical storage",
                 grid=(1024, 1024), kind="gaussian", ell=0.1, rank=32, b=32, leaf=64),
    "cfg2b1": dict(workload="cfg2 structure with 1 vector (HBM-bound variant)", grid=(1024, 1024),
                   kind="gaussian", ell=0.1, rank=32, b=1, leaf=64),
    # BASELINE.json configs[0] structure (hgemv part)
    "cfg1": dict(workload="2D exponential-kernel H2 hgemv N=16384 (128^2), leaf 64, rank 32, 1 vector",
                 grid=(128, 128), kind="exponential", ell=0.2, rank=32, b=1, leaf=64,
                 l2_flush=True),   # the 85 MB payload fits in the 126 MB L2
    # BASELINE.json configs[0]'s build: peel_construct over DenseOperator of the 128^2 exponential kernel
    # (eps 1e-4, max_rank 0), the matrix resident in HBM as the black box
    "cfg1build": dict(workload="HARA peel_construct(DenseOperator(K)) of the 2D exponential kernel K=exp(-|x-y|/0.2) "
                               "on the 128^2 grid (N=16384, dense 2.1 GB), strong admissibility eta=1, leaf 64, eps 1e-4, "
                               "max_rank 0, PeelConfig defaults (b=16, p=10, seed 42)",
                      grid=(128, 128), kind="exponential", ell=0.2, leaf=64, eps=1e-4, hara=True, dense=True),
    # BASELINE.json configs[2]: HARA from a black-box matvec of a diffusion Hessian: the reference's own
    # "diff1d-262144" oracle (registry.hpp:104-124; misfit + TV Hessian at the target density, two
    # Crank-Nicolson marches per source per application) with steps=64 as SURVEY §9.3 recommends,
    # applied on the device (paper_2003_10173_b200/csrc/diffusion1d.cu)
    "cfg3": dict(workload="HARA peel_construct from the black-box diffusion Hessian diff1d-262144 (registry.hpp:104-124, "
                          "steps=64, misfit+TV, 3 sources, 8 receivers; operator marched on the B200), N=2^18, "
                          "weak admissibility, leaf 32, eps 1e-6, PeelConfig defaults (b=16, p=10)",
                 grid=(262144,), pde=True, steps=64, leaf=32, eps=1e-6, hara=True, sample_n=16384),
    # the earlier analytic proxy: the heat propagator F = exp(T*Laplacian) is a Gaussian convolution, so
    # the misfit Hessian F^T F of a fully observed 1D diffusion inverse problem is a Gaussian kernel,
    # applied as a rank-32 H^2 (hgemv) on the same weak 1D tree
    "cfg3k": dict(workload="HARA peel_construct from a black-box matvec, 1D diffusion-Hessian proxy "
                           "(Gaussian heat-kernel F^T F, ell=0.05, applied as a rank-32 H^2), N=2^18, "
                           "weak admissibility, leaf 32, eps 1e-6, PeelConfig defaults (b=16, p=10)",
                  grid=(262144,), kind="gaussian", ell=0.05, rank=32, leaf=32, eps=1e-6, hara=True,
                  sample_n=16384),
    # BASELINE.json configs[4]: recompression + low-rank update, then hierarchical Newton-Schulz on a
    # regularised Hessian proxy at N=2^16: SURVEY §9.4's surface256 (the minimal-surface Hessian of the paper's
    # own testbed, at 256^2) built by HARA, + alpha I (alpha = 10: with alpha <= 3 the
    # reference's own driver stalls or diverges at residual 1e-6 -- DESIGN §7), a rank-8 symmetric update
    "cfg5": dict(workload="recompress(1e-8) + rank-8 low_rank_update + hierarchical Newton-Schulz (dynamic threshold "
                          "schedule from 1e-2, residual 1e-6) of the regularised minimal-surface Hessian surface256 "
                          "(N=2^16, strong admissibility, leaf 64; HARA of the sparse device black box at eps 1e-8) "
                          "+ 10 I",
                 grid=(65536,), surface=256, alpha=10.0, eps=1e-6, inversion=True, update_rank=8, sample_surface=64),
    # BASELINE.json configs[3] at P=1
    "cfg4": dict(workload="3D Matern-3/2 H2 hgemv N=2^21 (128^3 grid), leaf 64, rank 32, 64 vectors",
                 grid=(128, 128, 128), kind="matern32", ell=0.1, rank=32, b=64, leaf=64),
}

PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
def _fp64_peak():
    """FP64 tensor-path roofline denominator: profiles/fp64_peak.json (tools/measure_fp64_peak.py,
    DMMA m8n8k4 measured on this pool's B200 with SM clocks recorded), else the round-1 figure."""
    path = os.path.join(ROOT, "profiles", "fp64_peak.json")
    try:
        with open(path) as f:
            d = json.load(f)
        clk = d.get("clocks", {})
        return d["dmma_tflops"], (f"measured: tools/fp64_peak.cu DMMA m8n8k4 f64 on B200 at SM "
                                  f"{clk.get('sm_mhz')} MHz (max {clk.get('sm_max_mhz')}), profiles/fp64_peak.json")
    except (OSError, KeyError, ValueError):
        return 37.1, "measured round 1: tools/fp64_peak.cu DMMA m8n8k4 f64 (profiles/r01/fp64_peak.txt, no clock record)"


FP64_PEAK_TFLOPS, FP64_PEAK_SOURCE = _fp64_peak()


def ncu_traffic(config):
    """DRAM bytes per launch of the config's dominant kernel from its committed
    `ncu --set full` capture (tools/ncu_traffic.py -> profiles/ncu_traffic_<config>.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", f"ncu_traffic_{config}.json")) as f:
            d = json.load(f)
        return d["traffic_bytes_per_launch"], f"profiles/ncu_traffic_{config}.json ({d['kernel'][:60]}, {d['when']})"
    except (OSError, KeyError, ValueError):
        return None, None


def grid_points(shape):
    if len(shape) == 1:
        n = shape[0]
        return (-1.0 + 2.0 * np.arange(n) / (n - 1))[:, None]   # grid1d(n, -1, 1), test_support.hpp:12-16
    if len(shape) == 2:
        nx, ny = shape
        i = np.tile(np.arange(nx), ny)
        j = np.repeat(np.arange(ny), nx)
        return np.stack([i / (nx - 1), j / (ny - 1)], axis=1)
    nx, ny, nz = shape
    i = np.tile(np.arange(nx), ny * nz)
    j = np.tile(np.repeat(np.arange(ny), nx), nz)
    k = np.repeat(np.arange(nz), nx * ny)
    return np.stack([i / (nx - 1), j / (ny - 1), k / (nz - 1)], axis=1)


def hbm_peak():
    try:
        return float(json.load(open(PEAKS_FILE))["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        return 6650.0, "fallback B200_PROFILING.md"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self._started = threading.Event()
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            self._started.wait(timeout=3.0)   # sampling is live before the timed region starts
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())
            self._started.set()

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(names, f[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def free_port():
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def launch_ranks(args):
    """`--gpus N` without a torchrun environment: re-launch this command as N
    ranks under torch.distributed.run (one process per GPU, NCCL). Fails loudly
    when the node has fewer than N GPUs -- never falls back to one GPU."""
    if "WORLD_SIZE" in os.environ:
        world = int(os.environ["WORLD_SIZE"])
        if args.impl == "b200" and world != args.gpus:
            sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
        return
    if args.gpus <= 1 or args.impl == "reference":
        return   # the reference arm is the host CPU port: rank 0 alone does the work
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} requested but this node has {have} CUDA device(s); "
                 f"refusing to run (no single-GPU fallback)")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    print(f"bench.py: launching {args.gpus} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    sys.exit(subprocess.call(cmd))


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    pg = None
    if world > 1:
        import torch
        import torch.distributed as dist
        if args.impl != "reference":
            have = torch.cuda.device_count()
            if local >= have:
                sys.exit(f"bench.py: rank {rank} has LOCAL_RANK {local} but only {have} CUDA device(s)")
            torch.cuda.set_device(local)
        backend = "nccl" if args.impl != "reference" else "gloo"
        dist.init_process_group(backend=backend)
        pg = dist
        print(f"bench.py: rank {rank}/{world} on cuda:{local} backend={backend}", file=sys.stderr, flush=True)
    return world, rank, local, pg


def algorithmic_flops(m, bt, b):
    """Reference flop count of one hgemv: F = 2b(2 sum_leaf m k + 2 sum_nonroot k k_par
    + sum_adm k_r k_c + sum_dense m_r m_c), both orientations of every block; also the stage-5 part
    (dense near-field + leaf expansion)."""
    ct = bt.tree
    r, _ = m.ranks()
    r = r.astype(np.float64)
    size = (ct.end - ct.begin).astype(np.float64)
    leaves = ct.leaves
    nonroot = np.nonzero(ct.parent >= 0)[0]
    adm, dense = bt.admissible_leaves, bt.dense_leaves
    leaf_t = float(np.sum(size[leaves] * r[leaves]))
    xfer = float(np.sum(r[nonroot] * r[ct.parent[nonroot]]))
    coup = float(np.sum(r[bt.row[adm]] * r[bt.col[adm]]))
    dns = float(np.sum(size[bt.row[dense]] * size[bt.col[dense]]))
    total = 2.0 * b * (2 * leaf_t + 2 * xfer + coup + dns)
    stage5 = 2.0 * b * (leaf_t + dns)
    return total, stage5


def algorithmic_bytes(m, bt, b):
    """Compulsory HBM bytes of one hgemv: stored payload once, bases and transfers twice
    (up and down), x read and y written; from the structure, so it holds for sharded matrices too."""
    ct = bt.tree
    r, _ = m.ranks()
    r = r.astype(np.float64)
    size = (ct.end - ct.begin).astype(np.float64)
    leaves = ct.leaves
    nonroot = np.nonzero(ct.parent >= 0)[0]
    adm, dense = bt.admissible_leaves, bt.dense_leaves
    canon_a = adm[bt.row[adm] <= bt.col[adm]]
    canon_d = dense[bt.row[dense] <= bt.col[dense]]
    U = float(np.sum(size[leaves] * r[leaves]))
    E = float(np.sum(r[nonroot] * r[ct.parent[nonroot]]))
    S = float(np.sum(r[bt.row[canon_a]] * r[bt.col[canon_a]]))
    D = float(np.sum(size[bt.row[canon_d]] * size[bt.col[canon_d]]))
    return 8.0 * (2 * U + 2 * E + S + D + 2 * ct.n * b)


def stage5_roofline(args, m, n, b, F5, stages):
    """Roofline of the dominant launch (leaf expansion + dense near-field, stage 5): algorithmic flops of
    the reference for that stage (the kernel also applies U_t E_t, the folded finest downsweep step)."""
    dom = dict(stages[5])
    dom["kernel_gflop"] = dom["gflop"]
    dom["gflop"] = F5 / 1e9
    sizes = m.packed_sizes()
    dom["gbytes"] = (8.0 * (sizes[5] + sizes[0]) + 16.0 * n * b) / 1e9   # D and U once, x read, y written
    hbm, hbm_src = hbm_peak()
    ai = dom["gflop"] / max(dom["gbytes"], 1e-30)
    ridge = FP64_PEAK_TFLOPS * 1e3 / hbm
    if ai >= ridge:
        achieved = dom["gflop"] / (dom["ms"] / 1e3) / 1e3
        roof = {"bound": "tensor", "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": achieved / FP64_PEAK_TFLOPS, "peak_source": FP64_PEAK_SOURCE}
    else:
        achieved = dom["gbytes"] / (dom["ms"] / 1e3)
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                "peak_source": hbm_src}
    kname = ("seg_gemm_kernel<64,32,4,1,2,32,VEC,kModeY> (leaf expansion + dense near-field)" if b > 2 else
             "sym_pass64_kernel (dense near-field, each canonical block streamed once) + seg_gemm leaf expansion "
             "+ csr_sum")
    roof.update({"kernel": kname, "share_of_step": dom["ms"] / sum(s["ms"] for s in stages.values()),
                 "traffic": args.traffic, "traffic_source": args.traffic_source,
                 "traffic_over_algorithmic": (args.traffic / (dom["gbytes"] * 1e9)) if args.traffic else None,
                 "algorithmic_gflop": dom["gflop"], "algorithmic_gbytes": dom["gbytes"], "ms": dom["ms"]})
    return roof


def algorithmic_work(m, b, launches_stats=None):
    """F (flops) and B (bytes) of one hgemv per SURVEY §8(d)."""
    sizes = m.packed_sizes()   # U, E, V, F, S, D (doubles)
    n = m.tree.n
    B = 8.0 * (2 * (sizes[0] + sizes[2]) + 2 * (sizes[1] + sizes[3]) + sizes[4] + sizes[5] + 2 * n * b)
    return B


def run_b200(args, cfg, world, rank, local, dist):
    import torch
    import ctypes as C
    from paper_2003_10173_b200 import H2Matrix, build_block_tree, build_cluster_tree
    from paper_2003_10173_b200._lib import check, lib

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    b = args.b or cfg["b"]
    pts = grid_points(cfg["grid"])
    n = pts.shape[0]
    t0 = time.perf_counter()
    ct = build_cluster_tree(pts, cfg["leaf"], device=True)   # the same tree as the host builder, on the B200
    bt = build_block_tree(ct, ct, 1.0)
    t_tree = time.perf_counter() - t0
    t0 = time.perf_counter()
    # N > 1: every rank generates only its row-subtree shard's payload
    shard_mode = world > 1 or args.force_shard
    m = H2Matrix.kernel(bt, pts, cfg["kind"], cfg["ell"], cfg["rank"], shard=(world, rank) if shard_mode else None)
    t_gen = time.perf_counter() - t0
    rng = np.random.default_rng(42)
    x_host = torch.from_numpy(rng.standard_normal((b, n)))      # column-major n x b == row-major b x n
    X = x_host.to(dev)
    Y = torch.empty_like(X)
    stream = torch.cuda.current_stream(dev)
    sh = stream.cuda_stream
    sharded = None
    if shard_mode:
        # row-subtree sharding: each rank computes its subtree's rows; one NCCL all-to-all per hgemv
        from paper_2003_10173_b200.dist import ShardedHgemv
        sharded = ShardedHgemv(m, transport=args.transport, max_b=b)

    def step():
        if sharded is not None:
            sharded(X.t(), Y.t())
        else:
            check(lib.h2c_hgemv(m._h, 0, 0, n, b, X.data_ptr(), n, Y.data_ptr(), n, 1.0, 0.0, sh))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # per-launch stage timing + algorithmic work (roofline numerators)
    maxrec = 256
    cnt = C.c_int()
    st = np.zeros(maxrec, np.int32)
    ms = np.zeros(maxrec)
    fl = np.zeros(maxrec)
    by = np.zeros(maxrec)
    agg = {}
    for rep in range(max(3, min(args.steps, 10)) if sharded is None else 0):
        check(lib.h2c_hgemv_stage_times(m._h, 0, 0, n, b, X.data_ptr(), n, Y.data_ptr(), n, sh, maxrec,
                                        C.byref(cnt), st.ctypes.data_as(C.c_void_p), ms.ctypes.data_as(C.c_void_p),
                                        fl.ctypes.data_as(C.c_void_p), by.ctypes.data_as(C.c_void_p)))
        if rep == 0:
            continue
        for i in range(cnt.value):
            a = agg.setdefault(int(st[i]), [0.0, 0.0, 0.0, 0])
            a[0] += ms[i]
            a[1] += fl[i]
            a[2] += by[i]
            a[3] += 1
    nrep = max(3, min(args.steps, 10)) - 1
    stages = {k: {"ms": v[0] / nrep, "gflop": v[1] / nrep / 1e9, "gbytes": v[2] / nrep / 1e9,
                  "launches": v[3] // nrep} for k, v in agg.items()}
    F, F5 = algorithmic_flops(m, bt, b)
    Bbytes = algorithmic_bytes(m, bt, b)
    launches = m.launches(b) if sharded is None else sharded.plan.launches()

    # main timed region. A payload that fits in twice the L2 would be re-read from
    # L2 by back-to-back steps: then every step is preceded by an (untimed) write of
    # a buffer larger than L2 and timed on its own
    flush = None
    if cfg.get("l2_flush"):
        flush = torch.empty(FLUSH_BYTES // 8, dtype=torch.float64, device=dev)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        if flush is None:
            e0.record(stream)
            for _ in range(args.steps):
                step()
            e1.record(stream)
            torch.cuda.synchronize()
            elapsed = e0.elapsed_time(e1) / 1e3
        else:
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(args.steps)]
            for i in range(args.steps):
                flush.fill_(float(i))
                evs[i][0].record(stream)
                step()
                evs[i][1].record(stream)
            torch.cuda.synchronize()
            elapsed = sum(a.elapsed_time(z) for a, z in evs) / 1e3
    if dist:
        t = torch.tensor([elapsed], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t.item())
    t_step = elapsed / args.steps
    value = F / t_step / 1e9          # one hgemv of the whole matrix per step (all ranks together)
    gbs = Bbytes / t_step / 1e9

    if sharded is not None:
        # per-GPU roofline of the whole sharded step (stage timers run on the single-GPU path only)
        per_gpu = F / world / t_step / 1e12
        roof = {"bound": "tensor", "achieved": per_gpu, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": per_gpu / FP64_PEAK_TFLOPS, "peak_source": FP64_PEAK_SOURCE,
                "kernel": "whole sharded hgemv step per GPU (algorithmic flops / world / step time)",
                "traffic": None}
    else:
        roof = stage5_roofline(args, m, n, b, F5, stages)

    # end-to-end through the public host-buffer API (pinned x in, y out)
    xp = x_host.pin_memory()
    if sharded is not None:
        ob, orows = sharded.plan.owned_begin, sharded.plan.owned_rows
        perm = np.asarray(ct.perm)
        xop = torch.from_numpy(np.ascontiguousarray(x_host.numpy()[:, perm[ob:ob + orows]])).pin_memory()
        yops = [torch.empty_like(xop).pin_memory() for _ in range(3)]
        Xos = [xop.to(dev) for _ in range(3)]
        Yos = [torch.empty_like(Xos[0]) for _ in range(3)]
        # one plan (own workspace and exchange buffers) per rotating stream
        from paper_2003_10173_b200.dist import ShardedHgemv
        shs = [sharded] + [ShardedHgemv(m, transport=args.transport, max_b=b) for _ in range(2)]
    # rotating streams of the e2e leg (measured on cfg2: 2 -> 7.86, 3 -> 6.03-6.29, 4 -> 5.95-6.02,
    # 6 -> 6.04-6.07 ms per step; tools/ab/e2e_streams.py)
    NS = 4 if sharded is None else 3
    yps = [torch.empty_like(xp).pin_memory() for _ in range(NS)]
    streams = [torch.cuda.Stream(dev) for _ in range(NS)]

    def e2e_step(i):
        if sharded is None:
            # pipelined public API: step i on stream i % NS, so its H2D / D2H overlap the
            # neighbouring steps' hgemv (per-stream workspaces inside the library)
            check(lib.h2c_matvec_host_async(m._h, 0, 0, n, b, xp.data_ptr(), yps[i % NS].data_ptr(),
                                            streams[i % NS].cuda_stream))
        else:
            # each rank's slice of x / y (its owned rows, cluster order) lives in pinned host memory;
            # step i on stream i % 3 with its own plan, so copies overlap the neighbouring steps
            j = i % 3
            with torch.cuda.stream(streams[j]):
                Xos[j].copy_(xop, non_blocking=True)
                shs[j](Xos[j].t(), Yos[j].t(), owned=True)
                yops[j].copy_(Yos[j], non_blocking=True)

    def e2e_run(k):
        if flush is not None:   # L2-resident payload: flush, then time each call on its own
            tot = 0.0
            for i in range(k):
                flush.fill_(float(i))
                torch.cuda.synchronize()
                t = time.perf_counter()
                e2e_step(i)
                for st in streams:
                    st.synchronize()
                tot += time.perf_counter() - t
            return tot
        t = time.perf_counter()
        for i in range(k):
            e2e_step(i)
        for st in streams:
            st.synchronize()
        torch.cuda.synchronize()
        return time.perf_counter() - t

    # warm-up: three calls per stream (eager, graph capture, first replay), so the timed
    # region replays captured graphs on every stream
    tw = e2e_run(3 * NS if sharded is None else 6)
    if dist:
        dist.barrier()
    ke = max(4, min(args.steps, 20))
    te = e2e_run(ke) / ke
    if dist:
        t = torch.tensor([te], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        te = float(t.item())
    # the synchronous by-value call (H2D, hgemv, D2H, wait) for reference (single-GPU matrix only)
    ts = None
    if sharded is None:
        for _ in range(3):
            check(lib.h2c_matvec_host(m._h, 0, 0, n, b, xp.data_ptr(), yps[0].data_ptr()))
        t0 = time.perf_counter()
        for _ in range(3):
            check(lib.h2c_matvec_host(m._h, 0, 0, n, b, xp.data_ptr(), yps[0].data_ptr()))
        ts = (time.perf_counter() - t0) / 3
    io_rows = n if sharded is None else sharded.plan.owned_rows * world
    e2e = {"value": F / te / 1e9, "unit": "GFLOP/s", "ms_per_step": te * 1e3,
           "h2d_bytes_per_step": 8 * io_rows * b, "d2h_bytes_per_step": 8 * io_rows * b,
           "path": ("h2c_matvec_host_async on 4 rotating streams: per step pinned host x -> HBM, hgemv, "
                    "HBM -> pinned host y (copies of one step overlap the hgemv of the next)") if sharded is None else
                   "per rank, 3 rotating streams with a plan each: its owned rows of x (pinned host, cluster order) "
                   "-> HBM, sharded hgemv (NCCL all-to-all overlapped with the local near field), owned rows of y "
                   "-> pinned host",
           "warmup_s": tw,
           "sync_call": None if ts is None else {"value": F / ts / 1e9, "ms_per_step": ts * 1e3,
                                                 "path": "h2c_matvec_host (H2D, hgemv, D2H, wait; no overlap)"}}

    out = {
        "metric": "hgemv GFLOP/s (N=2^20, 32 vectors, fp64)" if args.config == "cfg2" else f"hgemv GFLOP/s ({args.config})",
        "value": value, "unit": "GFLOP/s", "gbytes_per_s": gbs, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (device-generated kernel matrix)",
        "config": hgemv_config(cfg, args, n, b, len(bt.admissible_leaves), len(bt.dense_leaves), world,
                               int(sharded.plan.recv_rows.sum()) * b * 8 if sharded is not None else None),
        "algorithmic": {"gflop_per_step": F / 1e9, "gbytes_per_step": Bbytes / 1e9},
        "stages": {str(k): v for k, v in sorted(stages.items())},
        "roofline": roof,
        "e2e": e2e,
        "gpu_launches": launches * args.steps,
        "clocks": clk.summary(),
        "setup_s": {"trees": t_tree, "generate": t_gen},
    }
    return out, (m, X, Y, n, b, F, ct, bt, pts)


def cpu_baseline_sample(args, ctx):
    """Oracle (CPU port of the reference) on a bounded sample of the same
    workload: the same H^2 payload, 2 of the b vectors, 1 thread."""
    import torch
    from oracle import pyoracle as O
    m, X, Y, n, b, F, ct, bt, pts = ctx
    bs = min(2, b)
    t0 = time.perf_counter()
    ref = O.Tree(pts, ct.leaf_size, 1.0, False)
    rr, _ = m.ranks()
    ora = O.H2.from_packed(ref, True, rr, None, m.download())
    t_load = time.perf_counter() - t0
    x = X[:bs].cpu().numpy().T
    t0 = time.perf_counter()
    y_ref = ora.matvec(x, threads=1)
    t = time.perf_counter() - t0
    y_gpu = Y[:bs].cpu().numpy().T
    relerr = float(np.linalg.norm(y_gpu - y_ref) / np.linalg.norm(y_ref))
    Fs = F * bs / b
    return {"value": Fs / t / 1e9, "unit": "GFLOP/s", "cores": 1, "kind": "port",
            "sample": f"full cfg matrix (same payload), {bs} of {b} vectors, 1 thread, {t:.1f} s",
            "seconds": t, "load_s": t_load, "parity_rel_err_full_size": relerr}


def hgemv_config(cfg, args, n, b, tree_adm, tree_dense, world, recv_bytes=None):
    """The `config` dict of an hgemv line (identical on the B200 and reference arms)."""
    return {"workload": cfg["workload"], "n": n, "vectors": b, "rank": cfg["rank"], "leaf": cfg["leaf"],
            "kernel": f"{cfg['kind']} ell={cfg['ell']}", "admissible_leaves": int(tree_adm),
            "dense_leaves": int(tree_dense),
            "parallelism": (f"row-subtree sharded x{world} (x-hat / x halos per hgemv: "
                            + ("P2P writes into the peers' receive buffers with device-side signals"
                               if getattr(args, "transport", "collective") == "peer" else "one NCCL all-to-all")
                            + f", {recv_bytes} B received by rank 0)") if recv_bytes is not None else "single GPU",
            "l2": ("L2 flushed before every timed step (write of a 256 MB buffer, untimed; each step timed on its own): "
                   "the payload fits in L2") if cfg.get("l2_flush") else
                  "inputs larger than L2 (payload > 2x the 126 MB L2, no flush needed)"}


def run_reference(args, cfg, world, rank):
    """--impl reference: the CPU restatement of the reference (oracle) on the host
    cores, same config/metric/payload; one step = one oracle hgemv over a
    bounded sample of the vectors: up to two vectors per host thread, all host
    threads; the step count is bounded so the arm finishes within a few minutes."""
    from oracle import pyoracle as O
    if rank != 0:
        return None
    b = args.b or cfg["b"]
    threads = max(1, os.cpu_count() or 1)
    bs = min(b, 2 * threads)
    pts = grid_points(cfg["grid"])
    n = pts.shape[0]
    t0 = time.perf_counter()
    tree = O.Tree(pts, cfg["leaf"], 1.0, False)
    # the same kernel H^2 as the B200 arm (host restatement of its generator, to rounding)
    h = O.H2.kernel(tree, cfg["kind"], cfg["ell"], cfg["rank"], threads)
    setup = time.perf_counter() - t0
    x = np.asfortranarray(np.random.default_rng(42).standard_normal((n, bs)))
    # algorithmic flops for bs vectors (SURVEY §8d formula)
    sizes = h.info()[2]
    adm = tree.adm
    dense = tree.dense
    kr, _ = h.ranks()
    sz = tree.end - tree.begin
    Fcol = 2 * (2 * sizes[0] + 2 * sizes[1])
    Fcol += 2 * float(np.sum(kr[tree.brow[adm]].astype(np.float64) * kr[tree.bcol[adm]]))
    Fcol += 2 * float(np.sum(sz[tree.brow[dense]].astype(np.float64) * sz[tree.bcol[dense]]))
    nth = min(threads, bs)
    t0 = time.perf_counter()
    h.matvec(x, threads=nth)   # first warm-up step (also sizes the step budget)
    t1 = time.perf_counter() - t0
    warm = max(1, min(args.warmup, int(30.0 / max(t1, 1e-3))))
    for _ in range(warm - 1):
        h.matvec(x, threads=nth)
    steps = max(2, min(args.steps, int(150.0 / max(t1, 1e-3))))
    ts = []
    for _ in range(steps):
        t0 = time.perf_counter()
        h.matvec(x, threads=nth)
        ts.append(time.perf_counter() - t0)
    t = sum(ts) / len(ts)
    v = Fcol * bs / t / 1e9
    return {"impl": "reference", "metric": "hgemv GFLOP/s (N=2^20, 32 vectors, fp64)" if args.config == "cfg2"
            else f"hgemv GFLOP/s ({args.config})", "value": v, "unit": "GFLOP/s", "n_gpus": world,
            "steps": steps, "warmup": warm, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (the B200 arm's kernel H^2: host restatement of its generator)",
            "config": hgemv_config(cfg, args, n, b, len(tree.adm), len(tree.dense), 1),
            "cpu_baseline": {"value": v, "unit": "GFLOP/s", "cores": nth, "kind": "port",
                             "sample": f"{bs} of {b} vectors per step ({bs // nth} per host thread, {nth} threads), "
                                       f"oracle restatement of the reference's matvec (h2_matrix.hpp:246-305; its "
                                       f"GEMM beats the Eigen-shim build of the reference's own headers by ~25%, so "
                                       f"the faster CPU arm is reported); {steps} steps (bounded to ~150 s)"},
            "e2e": {"value": v, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "setup_s": setup}


def hara_problem(cfg, n):
    from paper_2003_10173_b200 import Admissibility, H2Matrix, build_block_tree, build_cluster_tree
    pts = grid_points((n,))
    ct = build_cluster_tree(pts, cfg["leaf"])
    bt = build_block_tree(ct, ct, 1.0, Admissibility.weak)
    src = H2Matrix.kernel(bt, pts, cfg["kind"], cfg["ell"], cfg["rank"])
    return pts, ct, bt, src


def dense_kernel(cfg):
    """(points, dense kernel matrix as a column-major host array) of a dense-black-box config."""
    import torch
    pts = grid_points(cfg["grid"])
    p = torch.from_numpy(pts)
    if torch.cuda.is_available():
        p = p.cuda()
    r = torch.cdist(p, p)
    k = torch.exp(-r / cfg["ell"]) if cfg["kind"] == "exponential" else torch.exp(-(r / cfg["ell"]) ** 2)
    return pts, np.asfortranarray(k.cpu().numpy())   # symmetric: C and F order hold the same numbers


def hara_operator(cfg, n):
    """(black-box operator, block tree, keep-alive) of a HARA config."""
    from paper_2003_10173_b200 import (Admissibility, DenseOperator, H2Operator, build_block_tree, build_cluster_tree,
                                       make_oracle)
    if cfg.get("dense"):
        pts, a = dense_kernel(cfg)
        ct = build_cluster_tree(pts, cfg["leaf"])
        bt = build_block_tree(ct, ct, 1.0, Admissibility.strong)
        return DenseOperator(a, True), bt, (pts, a)
    if cfg.get("pde"):
        o = make_oracle(f"diff1d-{n}", {"steps": str(cfg["steps"]), "leaf": str(cfg["leaf"])})
        return o.op, o.default_block_tree(), o
    pts, ct, bt, src = hara_problem(cfg, n)
    return H2Operator(src), bt, src


def hara_roofline():
    """The construction's batched kernels from their committed ncu captures (not live: one
    capture per kernel, tools/round_evidence.sh). They are small batched problems, latency-bound;
    the build is bounded by the black-box operator and the per-panel decisions."""
    import re
    out = {"bound": "tensor", "unit": "TFLOP/s", "peak": FP64_PEAK_TFLOPS, "peak_source": FP64_PEAK_SOURCE,
           "live": False, "per_kernel": []}
    for k in ("bgemm_kernel", "qr_kernel", "jacobi_kernel"):
        f = os.path.join(ROOT, "profiles", "r02", f"ncu_full_hara_{k}_r02.txt")
        if not os.path.exists(f):
            continue
        txt = open(f).read()

        def num(name, txt=txt):
            m = re.search(re.escape(name) + r"\s*=\s*([0-9.eE+-]+)\s*(\S*)", txt)
            return (float(m.group(1)), m.group(2)) if m else (None, "")
        dur, du = num("gpu__time_duration.sum")
        sec = dur * {"us": 1e-6, "ms": 1e-3, "ns": 1e-9, "s": 1.0}.get(du, 1e-6) if dur else None
        ops, _ = num("sm__ops_path_tensor_src_fp64.sum")
        fp64, _ = num("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active")
        dmma, _ = num("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active")
        grid, _ = num("launch__grid_size")
        ent = {"kernel": k, "duration_us": None if sec is None else sec * 1e6, "grid": grid,
               "dmma_pipe_active_pct": dmma, "fp64_pipe_active_pct": fp64, "source": os.path.relpath(f, ROOT)}
        if ops and sec:
            ent["achieved_tflops"] = ops / sec / 1e12
            ent["frac"] = ent["achieved_tflops"] / FP64_PEAK_TFLOPS
        out["per_kernel"].append(ent)
    if out["per_kernel"] and "achieved_tflops" in out["per_kernel"][0]:
        out["kernel"] = "bgemm_kernel (the construction's DMMA batched GEMM)"
        out["achieved"] = out["per_kernel"][0]["achieved_tflops"]
        out["frac"] = out["per_kernel"][0]["frac"]
    return out


def run_hara(args, cfg, world, rank, local, dist):
    """cfg3: HARA build time on the B200 (one step = one peel_construct)."""
    import torch
    from paper_2003_10173_b200 import PeelConfig, estimate_relative_error, peel_construct
    torch.cuda.set_device(local)
    n = int(np.prod(cfg["grid"]))
    op, bt, keep = hara_operator(cfg, n)
    rngs = {"device": 1, "reference": 0}
    pc = PeelConfig(eps=cfg["eps"], rng=rngs[args.hara_rng])
    for _ in range(max(1, min(args.warmup, 1))):
        peel_construct(op, bt, pc)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    steps = max(1, min(args.steps, 3))
    import ctypes as C
    from paper_2003_10173_b200._lib import lib as _l
    _l.h2b_plan_build_ms.restype = C.c_double
    _l.h2b_plan_build_ms.argtypes = [C.c_int]
    _l.h2b_plan_sync_ms.restype = C.c_double
    _l.h2b_plan_sync_ms.argtypes = [C.c_int]
    _l.h2b_kernel_launches.restype = C.c_longlong
    _l.h2b_kernel_launches.argtypes = [C.c_int]
    times, opms, launches = [], [], []
    with ClockSampler(local) as clk:
        for _ in range(steps):
            op.reset_counter()
            torch.cuda.synchronize()
            _l.h2b_plan_build_ms(1)
            _l.h2b_plan_sync_ms(1)
            _l.h2b_plan_parts_ms((C.c_double * 4)(), 1)
            _l.h2b_kernel_launches(1)
            t0 = time.perf_counter()
            res = peel_construct(op, bt, pc)
            torch.cuda.synchronize()
            times.append(time.perf_counter() - t0)
            launches.append(int(_l.h2b_kernel_launches(0)))
            opms.append(res.op_ms)
    t = statistics.median(times)
    if dist:
        tt = torch.tensor([t], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
    # one more build with the phase timers draining the stream at each phase end
    # (device-accurate phase split; not part of the timed steps)
    _l.h2b_hara_phase_sync(1)
    _l.h2b_hara_phase_reset()
    _l.h2b_plan_build_ms(1)
    _l.h2b_plan_sync_ms(1)
    _l.h2b_plan_parts_ms((C.c_double * 4)(), 1)
    t0 = time.perf_counter()
    peel_construct(op, bt, pc)
    torch.cuda.synchronize()
    t_phased = time.perf_counter() - t0
    _l.h2b_hara_phase_sync(0)
    plan_ms = _l.h2b_plan_build_ms(0)
    plan_sync_ms = _l.h2b_plan_sync_ms(0)
    parts = (C.c_double * 4)()
    _l.h2b_plan_parts_ms(parts, 0)
    ph = (C.c_double * 16)()
    _l.h2b_hara_phase_ms(ph, 16)
    phases = dict(zip(["rng", "op_apply", "residual_hgemv", "absorb", "transposed_pass", "local_updates",
                       "recompress", "dense_leaves", "orthogonalize_all", "truncation_bases", "projection"],
                      [round(v / 1e3, 4) for v in ph]))
    phases["hgemv_plan_builds"] = round(plan_ms / 1e3, 4)
    phases["hgemv_plan_builds_device_sync"] = round(plan_sync_ms / 1e3, 4)
    phases["hgemv_plan_builds_split"] = {"task_lists": round(parts[0] / 1e3, 4), "ue_products": round(parts[1] / 1e3, 4),
                                         "uploads": round(parts[2] / 1e3, 4), "count": int(parts[3])}
    phases["all_steps_s"] = [round(v, 4) for v in times]
    phases["phased_build_s"] = round(t_phased, 4)
    err = estimate_relative_error(op, res.matrix)
    prof = [int(v) for v in res.matrix.rank_profile()]
    data = ("synthetic: the reference's diff1d oracle (target density, Ricker sources) marched on the device"
            if cfg.get("pde") else "synthetic (device-generated kernel H^2 black box)")
    out = {"metric": hara_metric(cfg), "value": t, "unit": "s", "n_gpus": world,
           "steps": steps, "warmup": 1, "ms_per_step": t * 1e3, "higher_is_better": False, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64", "data": data,
           "config": {"workload": cfg["workload"], "n": n, "eps": cfg["eps"], "rng": args.hara_rng,
                      "parallelism": f"replicas x{world}" if world > 1 else "single GPU"},
           "hara": {"op_s": statistics.median(opms) / 1e3, "construction_s": t - statistics.median(opms) / 1e3,
                    "samples": res.stats.total, "relative_error_2norm": err, "rank_profile": prof,
                    "level_samples": [lv.samples for lv in res.stats.levels], "phases_s": phases},
           "gpu_launches": int(statistics.median(launches)) * steps,
           "gpu_launches_per_build": int(statistics.median(launches)),
           "roofline": hara_roofline(),
           "clocks": clk.summary()}
    if cfg.get("pde"):
        out["hara"]["pde_solves"] = keep.diffusion.pde_solves()
    if cfg.get("dense"):
        out["data"] = "synthetic: the dense kernel matrix generated on the device, applied as the black box from HBM"
    return out


def hara_metric(cfg):
    n = int(np.prod(cfg["grid"]))
    return f"HARA build time (N={n}, tol {cfg['eps']:g})"


def inversion_problem(grid, cfg):
    """(A0 = HARA of the surface<grid> Hessian at eps 1e-8 with the reference stream, the rank-8 factor)."""
    from paper_2003_10173_b200 import PeelConfig, build_block_tree, build_cluster_tree, make_oracle, peel_construct
    o = make_oracle(f"surface{grid}")
    ct = build_cluster_tree(o.points, o.leaf)
    bt = build_block_tree(ct, ct, o.eta, o.mode)
    a0 = peel_construct(o.op, bt, PeelConfig(eps=1e-8, rng=0)).matrix
    n = o.op.dim()
    X = 0.1 * np.random.default_rng(7).standard_normal((n, cfg["update_rank"]))
    return o, a0, X


def inversion_step(a0, X, cfg, pc):
    """recompress(A0 + alpha I) + low_rank_update + h_newton_schulz from the scaled identity."""
    import torch
    from paper_2003_10173_b200 import (ThresholdSchedule, h_newton_schulz, low_rank_update, recompress,
                                       scaled_identity_start)
    t = {}
    t0 = time.perf_counter()
    m = recompress(a0, 1e-12)   # a copy to shift (the shift is in place)
    m.add_diagonal(cfg["alpha"])
    ar = recompress(m, 1e-8)
    t["recompress"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    au = low_rank_update(ar, X, X, 1e-8)
    t["low_rank_update"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    x0 = scaled_identity_start(au)
    try:
        res = h_newton_schulz(au, x0, ThresholdSchedule(dynamic=True), cfg["eps"], pc)
    except Exception as e:
        tr = getattr(e, "trace", None)
        rows = [(r.iter, r.residual, r.eps_k, r.samples) for r in tr.rows] if tr else []
        raise RuntimeError(f"NS failed: {e}; trace {rows}") from e
    torch.cuda.synchronize()
    t["newton_schulz"] = time.perf_counter() - t0
    return t, res, au


def run_inversion(args, cfg, world, rank, local, dist):
    """cfg5: one step = recompress + low-rank update + hierarchical Newton-Schulz to residual eps."""
    import torch
    from paper_2003_10173_b200 import PeelConfig, residual_norm
    torch.cuda.set_device(local)
    t0 = time.perf_counter()
    o, a0, X = inversion_problem(cfg["surface"], cfg)
    setup = time.perf_counter() - t0
    n = o.op.dim()
    pc = PeelConfig(eps=cfg["eps"], rng=1)
    inversion_step(a0, X, cfg, pc)
    import ctypes as C
    from paper_2003_10173_b200._lib import lib as _l
    _l.h2b_kernel_launches.restype = C.c_longlong
    _l.h2b_kernel_launches.argtypes = [C.c_int]
    times, launches = [], []
    with ClockSampler(local) as clk:
        for _ in range(max(1, min(args.steps, 2))):
            _l.h2b_kernel_launches(1)
            t, res, au = inversion_step(a0, X, cfg, pc)
            launches.append(int(_l.h2b_kernel_launches(0)))
            times.append(t)
    tot = [sum(t.values()) for t in times]
    i = int(np.argsort(tot)[len(tot) // 2])
    rows = res.trace.rows
    return {"metric": inversion_metric(cfg), "value": tot[i], "unit": "s", "n_gpus": world,
            "steps": len(tot), "warmup": 1, "ms_per_step": tot[i] * 1e3, "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: the minimal-surface Hessian black box (device sparse solves), HARA-compressed; "
                    "random rank-8 update",
            "config": {"workload": cfg["workload"], "n": n, "alpha": cfg["alpha"], "parallelism": "single GPU"},
            "inversion": {"phases_s": {k: round(v, 4) for k, v in times[i].items()},
                          "iterations": len(rows), "converged": res.trace.converged,
                          "final_residual": res.trace.final_residual,
                          "residual_check": residual_norm(au, res.X),
                          "samples": res.trace.total_samples(),
                          "rows": [(r.iter, r.residual, r.eps_k, r.samples, round(r.wall_seconds, 4)) for r in rows],
                          "rank_profile": [int(v) for v in res.X.rank_profile()], "setup_s": setup},
            "gpu_launches": int(sum(launches)), "gpu_launches_per_step": launches,
            "clocks": clk.summary()}


def inversion_metric(cfg):
    return f"NS inversion time (N={cfg['grid'][0]}, residual {cfg['eps']:g})"


def cpu_baseline_inversion(args, cfg):
    """The reference's own h_newton_schulz (oracle/_ref: inversion.hpp compiled from its headers, on the
    host) on the same recipe at the bounded size surface<sample_surface>; the B200 on the same sample."""
    import torch
    from paper_2003_10173_b200 import PeelConfig, ThresholdSchedule, h_newton_schulz, low_rank_update, recompress
    M, kind = ref_module()
    g = cfg["sample_surface"]
    o, a0, X = inversion_problem(g, cfg)
    m = recompress(a0, 1e-12)
    m.add_diagonal(cfg["alpha"])
    au = low_rank_update(recompress(m, 1e-8), X, X, 1e-8)
    rr, _ = au.ranks()
    tree = M.Tree(np.asarray(o.points), o.leaf, o.eta, o.mode != 0)
    ha = M.H2.from_packed(tree, True, rr, None, au.download())
    t0 = time.perf_counter()
    _, rows, final, conv = ha.h_inverse(cfg["eps"], dynamic=True)
    tc = time.perf_counter() - t0
    t0 = time.perf_counter()
    from paper_2003_10173_b200 import scaled_identity_start
    res = h_newton_schulz(au, scaled_identity_start(au), ThresholdSchedule(dynamic=True), cfg["eps"],
                          PeelConfig(eps=cfg["eps"], rng=0))
    torch.cuda.synchronize()
    tg = time.perf_counter() - t0
    same = [int(r[3]) for r in rows] == [r.samples for r in res.trace.rows]
    return {"value": tc, "unit": "s", "cores": 1, "kind": kind,
            "sample": f"the same recipe at N={g * g} (surface{g}): the reference's h_newton_schulz "
                      f"({'compiled from its headers' if kind == 'reference' else 'restatement'}, single-threaded): "
                      f"{len(rows)} iterations, converged {conv}, final residual {final:.2e}; B200 on the same "
                      f"sample with the reference RNG stream: {tg:.2f} s, {len(res.trace.rows)} iterations",
            "b200_same_sample_s": tg, "speedup_same_sample": tc / tg, "same_trace_samples": same}


def ref_module():
    """The reference's own compiled code (oracle/_ref) when present, else the restatement."""
    try:
        from oracle import pyref as M
        return M, "reference"
    except Exception:
        from oracle import pyoracle as M
        return M, "port"


def cpu_hara_build(cfg, n, threads):
    """One peel_construct on the CPU of the same problem: (seconds, samples,
    operator seconds[, extra]). Dense configs run the reference's own compiled
    construction (oracle/_ref) around a threaded dense black box."""
    from oracle import pyoracle as O
    if cfg.get("dense"):
        M, kind = ref_module()
        pts, a = dense_kernel(cfg)
        ref = M.Tree(pts, cfg["leaf"], 1.0, False)
        t0 = time.perf_counter()
        h, st, ops = M.peel_dense_threads(ref, a, True, eps=cfg["eps"], threads=threads)
        t = time.perf_counter() - t0
        prof = np.zeros(ref.depth + 1, np.int64)
        np.maximum.at(prof, ref.level, h.ranks()[0])
        return t, st["total"], ops, {"kind": kind, "level_samples": st["level_samples"],
                                     "rank_profile": prof.tolist()}
    if cfg.get("pde"):
        d = O.Diff1D(n=n, steps=cfg["steps"])
        ref = O.Tree(d.points(), cfg["leaf"], 1.0, True)
        t0 = time.perf_counter()
        h, tot, ops = d.peel(ref, eps=cfg["eps"], threads=threads)
        t = time.perf_counter() - t0
        prof = np.zeros(ref.depth + 1, np.int64)
        np.maximum.at(prof, ref.level, h.ranks()[0])
        return t, tot, ops, {"kind": "port", "level_samples": d.last_stats["level_samples"],
                             "rank_profile": prof.tolist()}
    pts, ct, bt, src = hara_problem(cfg, n)
    ref = O.Tree(pts, cfg["leaf"], 1.0, True)
    rr, _ = src.ranks()
    osrc = O.H2.from_packed(ref, True, rr, None, src.download())
    t0 = time.perf_counter()
    _, tot = O.peel_h2(ref, osrc, eps=cfg["eps"])
    return time.perf_counter() - t0, tot, None, {"kind": "port"}


def cpu_baseline_hara(args, cfg):
    """The oracle (restated reference) on a bounded sample: the same problem
    at N = sample_n, next to the B200 on the same sample."""
    import torch
    from paper_2003_10173_b200 import PeelConfig, peel_construct
    if cfg.get("dense"):   # the full build (about a minute on the host cores): no smaller sample of this config
        threads = os.cpu_count()
        n = int(np.prod(cfg["grid"]))
        tc, tot, ops, ex = cpu_hara_build(cfg, n, threads)
        return {"value": tc, "unit": "s", "cores": threads, "kind": ex["kind"],
                "sample": f"the full N={n} build, 1 step ({'the reference construction compiled from its headers' if ex['kind'] == 'reference' else 'oracle restatement'}, "
                          f"single-threaded as written, around a dense black box applied on {threads} threads): "
                          f"{tot} samples, operator applies {ops:.1f} s",
                "level_samples": ex["level_samples"], "rank_profile": ex["rank_profile"]}
    n = cfg["sample_n"]
    threads = os.cpu_count() if cfg.get("pde") else 1
    tc, tot, ops, _ = cpu_hara_build(cfg, n, threads)
    op, bt, keep = hara_operator(cfg, n)
    peel_construct(op, bt, PeelConfig(eps=cfg["eps"], rng=0))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = peel_construct(op, bt, PeelConfig(eps=cfg["eps"], rng=0))
    torch.cuda.synchronize()
    tg = time.perf_counter() - t0
    opnote = f" (operator applies {ops:.2f} s on {threads} threads)" if ops is not None else ""
    return {"value": tc, "unit": "s", "cores": threads, "kind": "port",
            "sample": f"same problem at N={n} (oracle restatement): {tc:.2f} s{opnote}, {tot} samples; "
                      f"B200 on the same sample with the reference RNG stream: {tg:.3f} s, {res.stats.total} samples",
            "b200_same_sample_s": tg, "speedup_same_sample": tc / tg}


def reference_hara(args, cfg, world):
    """--impl reference for HARA configs. cfg3 (diffusion Hessian): the full
    N=2^18 build on the CPU restatement with every host thread applying the
    operator (the reference's construction is single-threaded); one step.
    cfg3k: the bounded N=sample_n sample."""
    if cfg.get("pde"):
        n = cfg["grid"][0]
        threads = os.cpu_count()
        t, tot, ops, ex = cpu_hara_build(cfg, n, threads)
        cb = {"value": t, "unit": "s", "cores": threads, "kind": "port",
              "sample": f"the full N={n} build, 1 step: {tot} samples, operator applies {ops:.1f} s on {threads} "
                        f"threads, construction {t - ops:.1f} s on 1 thread (oracle restatement of the construction "
                        f"and of the diffusion black box)",
              "level_samples": ex["level_samples"], "rank_profile": ex["rank_profile"]}
    else:
        cb = cpu_baseline_hara(args, cfg)
    return {"impl": "reference", "metric": hara_metric(cfg), "value": cb["value"], "unit": "s",
            "n_gpus": world, "steps": 1, "warmup": 0, "higher_is_better": False,
            "config": {"workload": cfg["workload"]}, "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="cfg2", choices=list(CONFIGS))
    ap.add_argument("--b", type=int, default=0, help="override the vector count")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--force-shard", action="store_true", help="use the sharded path even at N=1 (testing)")
    ap.add_argument("--transport", choices=["collective", "peer"], default="collective",
                    help="sharded exchange: torch.distributed all-to-all (NCCL) or P2P writes with device signals")
    ap.add_argument("--hara-rng", default="device", choices=["device", "reference"],
                    help="cfg3 Gaussian panels: device Philox (perf) or the reference host stream")
    ap.add_argument("--traffic", type=float, default=None,
                    help="dram bytes/launch of the dominant kernel (default: the committed ncu --set full capture "
                         "profiles/ncu_traffic_<config>.json written by tools/ncu_traffic.py)")
    args = ap.parse_args()
    # NCCL communicator setup (ranks, rings / NVLS) on stderr; stdout carries only the JSON line
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    launch_ranks(args)
    if args.warmup < 3 and args.impl == "b200":
        args.warmup = 3
    cfg = CONFIGS[args.config]
    args.traffic_source = "command line" if args.traffic is not None else None
    if args.traffic is None:
        args.traffic, args.traffic_source = ncu_traffic(args.config)
    world, rank, local, dist = dist_setup(args)
    if cfg.get("inversion"):
        if args.impl == "reference":
            if rank == 0:
                cb = cpu_baseline_inversion(args, cfg)
                print(json.dumps({"impl": "reference", "metric": inversion_metric(cfg), "value": cb["value"],
                                  "unit": "s", "n_gpus": world, "steps": 1, "warmup": 0, "higher_is_better": False,
                                  "config": {"workload": cfg["workload"], "sample": f"surface{cfg['sample_surface']}"},
                                  "cpu_baseline": cb,
                                  "e2e": {"value": cb["value"], "unit": "s", "h2d_bytes_per_step": 0,
                                          "d2h_bytes_per_step": 0}}), flush=True)
            return
        out = run_inversion(args, cfg, world, rank, local, dist)
        if rank == 0 and not args.no_cpu_baseline:
            try:
                out["cpu_baseline"] = cpu_baseline_inversion(args, cfg)
            except Exception as e:
                out["cpu_baseline"] = {"value": None, "error": repr(e)}
        if rank == 0:
            print(json.dumps(out), flush=True)
        return
    if cfg.get("hara"):
        if args.impl == "reference":
            if rank == 0:
                print(json.dumps(reference_hara(args, cfg, world)), flush=True)
            return
        out = run_hara(args, cfg, world, rank, local, dist)
        if rank == 0 and not args.no_cpu_baseline:
            try:
                out["cpu_baseline"] = cpu_baseline_hara(args, cfg)
                cb = out["cpu_baseline"]
                if "level_samples" in cb and args.hara_rng == "reference":
                    out["hara"]["same_samples_and_ranks_as_cpu"] = (
                        cb["level_samples"] == out["hara"]["level_samples"] and
                        cb["rank_profile"] == out["hara"]["rank_profile"])
            except Exception as e:
                out["cpu_baseline"] = {"value": None, "error": repr(e)}
        if rank == 0:
            print(json.dumps(out), flush=True)
        return
    if args.impl == "reference":
        out = run_reference(args, cfg, world, rank)
        if out is not None:
            print(json.dumps(out), flush=True)
        return
    out, ctx = run_b200(args, cfg, world, rank, local, dist)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            out["cpu_baseline"] = cpu_baseline_sample(args, ctx)
        except Exception as e:  # the baseline is reported, never fatal
            out["cpu_baseline"] = {"value": None, "error": repr(e)}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
