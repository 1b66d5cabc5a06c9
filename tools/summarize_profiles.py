"""Summarise a round's gpurun_out/pr_* captures into profiles/ (run locally).

    python tools/summarize_profiles.py r01

Writes profiles/<round>_bench.json, <round>_launches.csv (kernel rows only),
<round>_launch_shares.json, <round>_ncu_full_summary.json and traffic.json
(DRAM bytes per point for bench.py's roofline.traffic).  Point counts per
iteration come from the config-4 golden (the run is bit-exact to it).
"""

from __future__ import annotations

import csv
import json
import os
import subprocess
import sys
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Hit Rate", "L1/TEX Hit Rate",
        "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread",
        "Compute (SM) Throughput", "Issue Slots Busy", "Executed Ipc Active",
        "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp", "Branch Efficiency",
        "Mem Busy", "Max Bandwidth"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
       "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
       "lts__t_sectors_srcunit_tex_op_red.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
       "gpu__time_duration.sum",
       # the L1 ceiling of gather-bound kernels: wavefronts through the LSU data pipe
       "l1tex__data_pipe_lsu_wavefronts.sum",
       "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
       "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
       "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
       "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
       "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
       "lts__t_sectors.avg.pct_of_peak_sustained_elapsed",
       "sm__cycles_elapsed.avg", "smsp__issue_active.avg.pct_of_peak_sustained_elapsed"]


def ncu_csv(rep: str, page: str) -> list[list[str]]:
    r = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True, text=True)
    return list(csv.reader(r.stdout.splitlines()))


def summarize(rep: str) -> dict:
    out: dict = {}
    rows = ncu_csv(rep, "details")
    hdr = rows[0]
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") in WANT:
            out[d["Metric Name"]] = f'{d["Metric Value"]} {d.get("Metric Unit", "")}'.strip()
        if "Kernel Name" in d:
            out["kernel"] = d["Kernel Name"]
    rows = ncu_csv(rep, "raw")
    hdr, units = rows[0], rows[1]
    vals = dict(zip(hdr, rows[2]))
    unit = dict(zip(hdr, units))
    for k in RAW:
        if k in vals:
            out[k] = f"{vals[k]} {unit.get(k, '')}".strip()
    stalls = {k: float(vals[k].replace(",", "") or 0) for k in vals
              if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")}
    tot = sum(stalls.values()) or 1.0
    out["top_stalls_pct"] = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): round(100 * v / tot, 1)
                             for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:6]}
    return out


def to_bytes(s: str) -> float:
    v, *u = s.split()
    v = float(v.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    return v * scale.get(u[0] if u else "byte", 1)


def main():
    rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"
    # bench line
    line = [l for l in open(os.path.join(OUT, "pr_bench.json")) if l.startswith("{")][-1]
    bench = json.loads(line)
    json.dump(bench, open(os.path.join(PROF, f"{rnd}_bench.json"), "w"), indent=1)
    # launch list
    rows = list(csv.reader(l for l in open(os.path.join(OUT, "pr_launches.csv")) if not l.startswith("==")))
    hdr = rows[0]
    kept = [hdr] + [r for r in rows[1:] if len(r) == len(hdr)]
    with open(os.path.join(PROF, f"{rnd}_launches.csv"), "w", newline="") as f:
        csv.writer(f).writerows(kept)
    tot: "OrderedDict[str, float]" = OrderedDict()
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    for r in kept[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        tot[name] = tot.get(name, 0.0) + float(r[vi].replace(",", ""))
    s = sum(tot.values())
    shares = {k: round(v / s, 4) for k, v in sorted(tot.items(), key=lambda kv: -kv[1])}
    json.dump({"note": "ncu --metrics gpu__time_duration.sum --clock-control none of "
                       "`bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline` (cold-cache, "
                       "serialised: compare shares, not absolute times)",
               "total_ms": round(s / 1e6, 3), "shares": shares},
              open(os.path.join(PROF, f"{rnd}_launch_shares.json"), "w"), indent=1)
    # full captures
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "cfg4.json")))
    npts = [it["n_points"] for it in g["iterations"]]
    caps = {
        "hb_resample_emit": ("pr_emit_ring_kernel.ncu-rep", "emit of iteration 5 (reads N4, writes N5)",
                             npts[5]),
        "hb_advect_points": ("pr_advect_flat_kernel.ncu-rep", "advect of iteration 4 (N4 points)",
                             npts[4]),
        "hb_laplacian_count": ("pr_lapcount.ncu-rep",
                               "Laplacian + resample count of iteration 4 (N4 points)", npts[4]),
    }
    summary, traffic = {}, {}
    for api, (rep, what, n) in caps.items():
        p = os.path.join(OUT, rep)
        if not os.path.exists(p):
            continue
        sm = summarize(p)
        sm["capture"] = what
        sm["points"] = n
        rd = to_bytes(sm["dram__bytes_read.sum"])
        wr = to_bytes(sm["dram__bytes_write.sum"])
        sm["dram_bytes_per_point"] = round((rd + wr) / n, 2)
        summary[api] = sm
        traffic[api] = {"bytes_per_point": round((rd + wr) / n, 2), "source": f"{rnd} ncu --set full, {what}"}
    json.dump(summary, open(os.path.join(PROF, f"{rnd}_ncu_full_summary.json"), "w"), indent=1)
    json.dump(traffic, open(os.path.join(PROF, "traffic.json"), "w"), indent=1)
    print(json.dumps({"shares": shares, "traffic": traffic}, indent=1))


if __name__ == "__main__":
    main()
