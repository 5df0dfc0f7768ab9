"""Measure the FP64 roofline denominators on this B200 (DMMA m8n8k4 and DFMA
throughput, fp64 copy bandwidth) with SM clocks sampled during the run, and
write profiles/fp64_peak.json (read by bench.py). MEASURED_PEAKS.json (driver
written) carries HBM and bf16 only.

  python tools/measure_fp64_peak.py            # on the GPU box
"""
import json
import os
import re
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    exe = os.path.join(ROOT, "tools", "fp64_peak")
    src = os.path.join(ROOT, "tools", "fp64_peak.cu")
    if not os.path.exists(exe) or os.path.getmtime(exe) < os.path.getmtime(src):
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o", exe, src], check=True)
    from bench import ClockSampler
    with ClockSampler(0) as clk:
        out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout
    dmma = [float(v) for v in re.findall(r"DMMA threads=\d+: ([\d.]+)", out)]
    dfma = [float(v) for v in re.findall(r"DFMA threads=\d+: ([\d.]+)", out)]
    copy = [float(v) for v in re.findall(r"copy: ([\d.]+)", out)]
    res = {"dmma_tflops": max(dmma), "dfma_tflops": max(dfma), "fp64_copy_gbs": max(copy),
           "how": "tools/fp64_peak.cu: mma.sync m8n8k4 f64 (DMMA) / fma f64 chains on every SM, "
                  "8 independent accumulators per warp, best of 3 block sizes; copy = 2 GiB read + write",
           "clocks": clk.summary(), "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
           "raw": out.strip().splitlines()}
    path = os.path.join(ROOT, "profiles", "fp64_peak.json")
    with open(path, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps({k: res[k] for k in ("dmma_tflops", "dfma_tflops", "fp64_copy_gbs", "clocks")}))


if __name__ == "__main__":
    main()
