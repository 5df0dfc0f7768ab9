"""One `ncu --set full` capture of a config's dominant hgemv kernel -> the
DRAM traffic per launch that bench.py reports as roofline.traffic
(profiles/ncu_traffic_<config>.json), plus the human-readable summary.

  python tools/ncu_traffic.py cfg2     # on the GPU box, after bench.py ran clean
"""
import csv
import io
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# dominant kernel per config (name regex for ncu) and how many matching launches to skip
# (past the warm-up and the stage-timed calls, into the steady state)
# (demangled-name regex, launches to skip, description)
TARGETS = {
    "cfg2": ("regex:seg_gemm_kernel", 30, 30, "seg_gemm kModeY (leaf expansion + dense near field): the longest captured launch"),
    "cfg4": ("regex:seg_gemm_kernel", 30, 30, "seg_gemm kModeY (leaf expansion + dense near field): the longest captured launch"),
    "cfg2b1": ("regex:sym_tma64_kernel|sym_pass64_kernel", 4, 2, "symmetric few-vector dense block pass"),
    "cfg1": ("regex:sym_tma64_kernel|sym_pass64_kernel", 4, 2, "symmetric few-vector dense block pass"),
}


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    name, skip, count, what = TARGETS[cfg]
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    rep = os.path.join(ROOT, "gpurun_out", f"ncu_traffic_{cfg}")
    cmd = ["ncu", "--set", "full", "--clock-control", "none", "--import-source", "on", "--kernel-name-base", "function",
           "--kernel-name", name, "--launch-skip", str(skip), "--launch-count", str(count), "-f", "-o", rep,
           sys.executable, os.path.join(ROOT, "bench.py"), "--config", cfg, "--steps", "3", "--warmup", "3",
           "--no-cpu-baseline"]
    subprocess.run(cmd, check=True, stdout=subprocess.DEVNULL)
    out = subprocess.run(["ncu", "-i", rep + ".ncu-rep", "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], dict(zip(rows[0], rows[1]))
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
             "nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9, "%": 1.0, "": 1.0}
    launches = []
    for row in rows[2:]:
        d = dict(zip(hdr, row))

        def num(k, d=d):   # to bytes / nanoseconds, whatever unit ncu chose for this column
            v = d.get(k, "")
            return float(v.replace(",", "")) * scale.get(units.get(k, ""), 1.0) if v else float("nan")
        launches.append({"kernel": d.get("Kernel Name", ""), "duration_ns": num("gpu__time_duration.sum"),
                         "dram_read_bytes": num("dram__bytes_read.sum"), "dram_write_bytes": num("dram__bytes_write.sum"),
                         "l2_hit_pct": num("lts__t_sector_hit_rate.pct"),
                         "dmma_pct": num("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active")})
    # the heaviest launch among the captured ones is the dominant kernel
    dom = max(launches, key=lambda r: r["duration_ns"])
    res = {"config": cfg, "kernel": dom["kernel"], "what": what,
           "traffic_bytes_per_launch": dom["dram_read_bytes"] + dom["dram_write_bytes"], "launch": dom,
           "captured": launches, "command": " ".join(cmd), "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    with open(os.path.join(ROOT, "profiles", f"ncu_traffic_{cfg}.json"), "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps({k: res[k] for k in ("config", "kernel", "traffic_bytes_per_launch")}))


if __name__ == "__main__":
    main()
