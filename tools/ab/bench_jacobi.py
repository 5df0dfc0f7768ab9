"""Microbenchmark of the batched Jacobi SVD (h2b_bench_jacobi): ms per call and sweeps."""
import ctypes as C
import os
import sys
sys.path.insert(0, os.getcwd())
from paper_2003_10173_b200._lib import lib  # noqa: E402
for n in [int(v) for v in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["64", "128"])]:
    st0 = (C.c_ulonglong * 5)()
    lib.h2b_jacobi_stats(st0)
    ms = C.c_double()
    lib.h2b_bench_jacobi(n, 100, 1, 3, C.byref(ms))
    st1 = (C.c_ulonglong * 5)()
    lib.h2b_jacobi_stats(st1)
    sw, pr = st1[0] - st0[0], st1[1] - st0[1]
    print(f"n={n}: {ms.value:.3f} ms per call of 100 problems, {sw / max(pr, 1):.2f} sweeps on average", flush=True)
