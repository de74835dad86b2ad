"""Summarise ncu captures into profiles/ (tracked). Usage:
    python profiles/summarize.py <report.ncu-rep> <name> [--launches launches.csv]
Writes profiles/<name>.json (key metrics of the captured fused-kernel launch, stall
breakdown, per-launch DRAM traffic) and, with --launches, the per-kernel share of the step
from the serialised launch list."""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_inst_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "smsp__warps_active.avg.per_cycle_active": "warps_per_scheduler",
    "launch__registers_per_thread": "registers",
    "smsp__inst_executed.sum": "warp_instructions",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum": "thread_dfma",
    "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum": "thread_dmul",
    "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum": "thread_dadd",
    "lts__t_bytes.sum": "l2_bytes",
    "sm__cycles_elapsed.avg.per_second": "sm_clock_hz",
}


def raw(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def to_base(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1e-3, "us": 1e-6,
             "ns": 1e-9, "s": 1, "hz": 1, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9}.get(unit, 1)
    return float(v.replace(",", "")) * scale


def summarize(report, name, launches=None, zones=None):
    h, u, rows = raw(report)
    res = {"report": os.path.basename(report), "kernels": []}
    for r in rows:
        k = {"name": r[h.index("Kernel Name")][:120]}
        for key, short in KEYS.items():
            if key in h:
                i = h.index(key)
                try:
                    k[short] = to_base(r[i], u[i])
                except ValueError:
                    pass
        stalls = {}
        for i, key in enumerate(h):
            if key.startswith("smsp__average_warps_issue_stalled_") and \
                    key.endswith("_per_issue_active.ratio"):
                try:
                    stalls[key[len("smsp__average_warps_issue_stalled_"):-len(
                        "_per_issue_active.ratio")]] = float(r[i])
                except ValueError:
                    pass
        k["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda x: -x[1])[:10])
        if zones:
            k["zones"] = zones
            k["dram_bytes_per_zone"] = (k.get("dram_read", 0) + k.get("dram_write", 0)) / zones
            fp64 = k.get("thread_dfma", 0) + k.get("thread_dmul", 0) + k.get("thread_dadd", 0)
            if fp64:
                k["fp64_thread_instr_per_zone(dfma+dmul+dadd)"] = fp64 / zones
        res["kernels"].append(k)
    if launches:
        res["launch_share"] = launch_share(launches)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), name + ".json")
    with open(path, "w") as f:
        json.dump(res, f, indent=1)
    return res


def launch_share(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    d = defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > vi:
            d[r[ki].split("(")[0][:80]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for k, v in d.items() if "dfma_peak" not in k and "dt_next" not in k)
    return {k: {"launches": len(v), "mean_ns": sum(v) / len(v),
                "share_of_step": (sum(v) / tot if ("dfma_peak" not in k and "dt_next" not in k)
                                  else None)}
            for k, v in d.items()}


if __name__ == "__main__":
    args = sys.argv[1:]
    lp = None
    zones = None
    if "--launches" in args:
        i = args.index("--launches")
        lp = args[i + 1]
        del args[i:i + 2]
    if "--zones" in args:
        i = args.index("--zones")
        zones = float(args[i + 1])
        del args[i:i + 2]
    print(json.dumps(summarize(args[0], args[1], lp, zones), indent=1))
