"""Aggregate H2_TRACE_SVD lines (la::bleft_svd per-step times) from stdin by problem shape."""
import collections
import sys

agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0, 0])
for line in sys.stdin:
    if not line.startswith("left_svd"):
        continue
    d = dict(kv.split("=") for kv in line.split()[1:])
    key = (int(d["mmax"]) // 16 * 16, int(d["cmax"]) // 256 * 256)
    a = agg[key]
    a[0] += 1
    a[1] += float(d["copy"])
    a[2] += float(d["qr"])
    a[3] += float(d["jacobi"])
    a[4] += int(d["problems"])
print("tot calls %d copy %.1f qr %.1f jacobi %.1f ms" % ((sum(v[0] for v in agg.values()),) +
                                                        tuple(sum(v[i] for v in agg.values()) for i in (1, 2, 3))))
for k, v in sorted(agg.items(), key=lambda kv: -(kv[1][2] + kv[1][3]))[:12]:
    print("m~%3d c~%4d: calls %4d copy %7.1f qr %7.1f jacobi %7.1f problems %6d" % (k[0], k[1], v[0], v[1], v[2], v[3], v[4]))
