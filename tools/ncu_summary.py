"""Summarise ncu captures for profiles/ (run here, no GPU needed).

  python tools/ncu_summary.py gpurun_out/prof_dense_cfg2_r01.ncu-rep [...]  > profiles/x.txt
  python tools/ncu_summary.py --launches gpurun_out/launches_cfg2_r01.csv   > profiles/y.txt
"""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "sm__ops_path_tensor_src_fp64.sum",
    "sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "lts__t_sector_hit_rate.pct",
    "launch__grid_size",
    "launch__block_size",
    "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic",
    "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem",
    "launch__waves_per_multiprocessor",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]


def summarise(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    print(f"== {rep}")
    for row in rows[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        print(f"kernel: {d.get('Kernel Name', '?')}")
        for k in KEYS:
            if k in d:
                print(f"  {k} = {d[k]} {u.get(k, '')}")
        stalls = []
        for k in hdr:
            if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio"):
                try:
                    v = float(d[k])
                except ValueError:
                    continue
                if v >= 0.1:
                    stalls.append((v, k.replace("smsp__average_warps_issue_stalled_", "").replace(
                        "_per_issue_active.ratio", "")))
        stalls.sort(reverse=True)
        print("  stalls (warps per issue): " + ", ".join(f"{n} {v:.2f}" for v, n in stalls))


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    recs = []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                recs.append((d["Kernel Name"], float(d["Metric Value"]), d.get("Metric Unit", "")))
    print(f"== {path}: {len(recs)} launches (cold-cache, serialised; compare shares)")
    for name, v, u in recs:
        print(f"{v:12.0f} {u:5s} {name[:110]}")


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        for p in sys.argv[2:]:
            launches(p)
    else:
        for p in sys.argv[1:]:
            summarise(p)
