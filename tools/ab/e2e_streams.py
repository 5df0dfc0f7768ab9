"""e2e (pinned host x -> h2c_matvec_host_async -> pinned host y) with S rotating streams, cfg2."""
import os
import sys
import time
sys.path.insert(0, os.getcwd())
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2003_10173_b200 import H2Matrix, build_block_tree, build_cluster_tree  # noqa: E402
from paper_2003_10173_b200._lib import check, lib  # noqa: E402
cfg = bench.CONFIGS["cfg2"]
pts = bench.grid_points(cfg["grid"])
n, b = pts.shape[0], 32
ct = build_cluster_tree(pts, 64, device=True)
bt = build_block_tree(ct, ct, 1.0)
m = H2Matrix.kernel(bt, pts, "gaussian", 0.1, 32)
xp = torch.randn(b, n, dtype=torch.float64).pin_memory()
for S in [int(v) for v in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["2", "3", "4"])] * 2:
    yps = [torch.empty(b, n, dtype=torch.float64).pin_memory() for _ in range(S)]
    streams = [torch.cuda.Stream() for _ in range(S)]
    for i in range(3 * S):
        check(lib.h2c_matvec_host_async(m._h, 0, 0, n, b, xp.data_ptr(), yps[i % S].data_ptr(), streams[i % S].cuda_stream))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    K = 20
    for i in range(K):
        check(lib.h2c_matvec_host_async(m._h, 0, 0, n, b, xp.data_ptr(), yps[i % S].data_ptr(), streams[i % S].cuda_stream))
    torch.cuda.synchronize()
    t = (time.perf_counter() - t0) / K
    print(f"streams={S}: {t * 1e3:.3f} ms per step", flush=True)
