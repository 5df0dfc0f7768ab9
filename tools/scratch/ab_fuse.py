"""A/B of the fused top-level sweeps (h2b_tune 11) for few-vector plans: ms per hgemv."""
import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2003_10173_b200 import H2Matrix, build_block_tree, build_cluster_tree
from paper_2003_10173_b200._lib import lib, check
import bench
ov = int(os.environ.get("OVERLAP", "1")); lib.h2b_tune(8, ov)
for cfg in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["cfg1", "cfg2"]):
    c = bench.CONFIGS[cfg]
    pts = bench.grid_points(c["grid"])
    n = pts.shape[0]
    ct = build_cluster_tree(pts, c["leaf"], device=True)
    bt = build_block_tree(ct, ct, 1.0)
    m = H2Matrix.kernel(bt, pts, c["kind"], c["ell"], c["rank"])
    s = torch.cuda.current_stream().cuda_stream
    for b in (1, 2):
        X = torch.randn(b, n, dtype=torch.float64, device="cuda")
        res, ys = {}, {}
        for knob in (0, 16, 64, 256, 1024, 0, 16, 64, 256, 1024):
            lib.h2b_tune(11, knob)
            Y = torch.empty_like(X)
            for _ in range(5):
                check(lib.h2c_hgemv(m._h, 0, 0, n, b, X.data_ptr(), n, Y.data_ptr(), n, 1.0, 0.0, s))
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(50):
                check(lib.h2c_hgemv(m._h, 0, 0, n, b, X.data_ptr(), n, Y.data_ptr(), n, 1.0, 0.0, s))
            e1.record(); torch.cuda.synchronize()
            res.setdefault(knob, []).append(e0.elapsed_time(e1) / 50)
            ys[knob] = Y.clone()
        line = " ".join(f"fuse{k}={min(v):.4f}" for k, v in res.items())
        d = max(float((ys[k] - ys[0]).abs().max() / ys[0].abs().max()) for k in ys)
        print(f"{cfg} b={b} overlap={ov}: {line} ms; max rel diff vs off {d:.2e}", flush=True)
lib.h2b_tune(11, 64)
