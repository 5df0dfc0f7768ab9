"""Symbolize and summarise a tools/sprof.c sample file.

  python tools/sprof_report.py gpurun_out/sprof.txt [--lib libh2b200] [--top 40]

Frames inside objects whose path contains --lib are symbolized with addr2line
against the local copy of that object (same build as the one profiled); other
frames are reported by object name. Prints self and inclusive sample counts.
"""
import argparse
import collections
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("file")
    ap.add_argument("--lib", default="libh2b200")
    ap.add_argument("--local", default=os.path.join(ROOT, "paper_2003_10173_b200", "lib", "libh2b200.so"))
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--callers", default=None, help="also list the nearest --lib callers of frames matching this")
    a = ap.parse_args()
    samples = [line.split() for line in open(a.file) if line.strip()]
    offs = set()
    for s in samples:
        for fr in s:
            obj, _, off = fr.rpartition("+")
            if a.lib in obj:
                offs.add(off)
    offs = sorted(offs)
    names = {}
    if offs:
        out = subprocess.run(["addr2line", "-f", "-C", "-e", a.local] + offs, capture_output=True, text=True).stdout
        lines = out.splitlines()
        for i, off in enumerate(offs):
            fn = lines[2 * i] if 2 * i < len(lines) else "?"
            names[off] = fn[:110]

    def label(fr):
        obj, _, off = fr.rpartition("+")
        if a.lib in obj:
            return names.get(off, "?")
        return "[" + os.path.basename(obj) + "]"

    self_c = collections.Counter()
    incl = collections.Counter()
    for s in samples:
        labs = [label(fr) for fr in s]
        if labs:
            self_c[labs[0]] += 1
        for lab in set(labs):
            incl[lab] += 1
    n = len(samples)
    print(f"{n} samples (1 ms of process CPU time each)")
    print("== self")
    for k, v in self_c.most_common(a.top):
        print(f"{v:7d} {100.0 * v / n:5.1f}%  {k}")
    print("== inclusive")
    for k, v in incl.most_common(a.top):
        print(f"{v:7d} {100.0 * v / n:5.1f}%  {k}")
    if a.callers:
        cal = collections.Counter()
        for s in samples:
            labs = [label(fr) for fr in s]
            hit = [i for i, lab in enumerate(labs) if a.callers in lab]
            if not hit:
                continue
            chain = [lab for lab in labs[hit[0] + 1:] if not lab.startswith("[") and "libcudart" not in lab][:3]
            cal[" <- ".join(c[:60] for c in chain)] += 1
        print(f"== callers of {a.callers}")
        for k, v in cal.most_common(a.top):
            print(f"{v:7d}  {k}")


if __name__ == "__main__":
    sys.exit(main())
