"""One HARA build (cfg3k problem) for an ncu launch list: how much of the build
is device time vs host time (run under ncu --metrics gpu__time_duration.sum)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2003_10173_b200 import PeelConfig, peel_construct

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3k"]
import numpy as np
op, bt, keep = bench.hara_operator(cfg, int(np.prod(cfg["grid"])))
pc = PeelConfig(eps=cfg["eps"], rng=int(sys.argv[2]) if len(sys.argv) > 2 else 1)
peel_construct(op, bt, pc)
torch.cuda.synchronize()
t = time.perf_counter()
res = peel_construct(op, bt, pc)
torch.cuda.synchronize()
print("build s", time.perf_counter() - t, "samples", res.stats.total)
