"""Summarise a tools/sprof.c sample file (SPROF_REAL=1: 1 ms of wall time per sample):
per sample, the innermost libh2b200 frame and whether the thread was inside the CUDA
driver (launch / copy / synchronisation) or running host code.

  python tools/wall_report.py gpurun_out/wall.txt.<pid> [--within peel_construct] [--top 40]"""
import argparse
import collections
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("file")
    ap.add_argument("--within", default=None)
    ap.add_argument("--top", type=int, default=40)
    a = ap.parse_args()
    lib = os.path.join(ROOT, "paper_2003_10173_b200", "lib", "libh2b200.so")
    samples = [line.split() for line in open(a.file) if line.strip()]
    offs = sorted({fr.rpartition("+")[2] for s in samples for fr in s if "libh2b200" in fr})
    out = subprocess.run(["addr2line", "-f", "-C", "-e", lib] + offs, capture_output=True, text=True).stdout.splitlines()
    names = {o: out[2 * i][:90] for i, o in enumerate(offs) if 2 * i < len(out)}

    def lab(fr):
        o, _, off = fr.rpartition("+")
        return names.get(off, "?") if "libh2b200" in o else "[" + os.path.basename(o) + "]"

    rows = [[lab(fr) for fr in s] for s in samples]
    if a.within:
        rows = [r for r in rows if any(a.within in x for x in r)]
    print(f"{len(rows)} samples (ms of wall time){' within ' + a.within if a.within else ''}")
    c = collections.Counter()
    incl = collections.Counter()
    for r in rows:
        h2 = [x for x in r if not x.startswith("[") and not x.startswith("cuda") and "libcudart" not in x]
        top = h2[0] if h2 else "(no libh2b200 frame)"
        drv = any("libcuda" in x for x in r[:8])
        c[(top, "driver" if drv else "host")] += 1
        for x in set(h2):
            incl[x] += 1
    print("== innermost libh2b200 frame, in the driver or in host code")
    for (k, w), v in c.most_common(a.top):
        print(f"{v:7d} {w:6s} {k}")
    print("== inclusive")
    for k, v in incl.most_common(a.top):
        print(f"{v:7d} {k}")


if __name__ == "__main__":
    main()
