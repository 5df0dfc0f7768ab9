"""A/B of the top chain (h2b_tune 12) on general plans: ms per hgemv."""
import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2003_10173_b200 import H2Matrix, build_block_tree, build_cluster_tree
from paper_2003_10173_b200._lib import lib, check
import bench
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
knobs = [int(v) for v in (sys.argv[3].split(",") if len(sys.argv) > 3 else ["0", "256", "1024", "4096"])]
c = bench.CONFIGS[cfg]
pts = bench.grid_points(c["grid"]); n = pts.shape[0]
ct = build_cluster_tree(pts, c["leaf"], device=True); bt = build_block_tree(ct, ct, 1.0)
m = H2Matrix.kernel(bt, pts, c["kind"], c["ell"], c["rank"])
s = torch.cuda.current_stream().cuda_stream
for b in [int(v) for v in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["32", "16"])]:
    X = torch.randn(b, n, dtype=torch.float64, device="cuda")
    res, ys = {}, {}
    for knob in knobs + knobs:
        lib.h2b_tune(12, knob)
        Y = torch.empty_like(X)
        for _ in range(4):
            check(lib.h2c_hgemv(m._h, 0, 0, n, b, X.data_ptr(), n, Y.data_ptr(), n, 1.0, 0.0, s))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            check(lib.h2c_hgemv(m._h, 0, 0, n, b, X.data_ptr(), n, Y.data_ptr(), n, 1.0, 0.0, s))
        e1.record(); torch.cuda.synchronize()
        res.setdefault(knob, []).append(e0.elapsed_time(e1) / 20)
        ys[knob] = Y.clone()
    same = all(torch.equal(ys[k], ys[knobs[0]]) for k in ys)
    print(f"{cfg} b={b}: " + " ".join(f"chain{k}={min(v):.4f}" for k, v in res.items()) + f" ms; bitwise equal {same}", flush=True)
lib.h2b_tune(12, 4096)
