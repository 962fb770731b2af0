#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) and one
`ncu --set full` report into profiles/:

  python tools/ncu_summary.py LAUNCHES.csv REPORT.ncu-rep TAG [MORE.ncu-rep ...]

writes profiles/<TAG>_launches.md (per-kernel time shares of the step),
profiles/<TAG>_ncu_full.md (key metrics per profiled kernel) and
profiles/ncu_traffic.json (DRAM bytes per launch for bench.py's roofline.traffic).
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_shared_mem",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio"]
SHORT = {"k_interp_push": "interp_push", "k_spread": "spread", "k_bin_count": "bin_count",
         "k_scatter_sorted": "scatter_sorted", "k_scatter_index": "scatter_index",
         "k_gather_sorted": "gather_sorted"}


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    unit = None
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", ""))
        unit = r[ui]
    return agg, unit


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        u = dict(zip(h, units))
        res.append((d["Kernel Name"], {k: (d.get(k), u.get(k)) for k in KEYS}))
    return res


def to_bytes(val, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return float(val.replace(",", "")) * scale


def main():
    lpath, rpath, tag = sys.argv[1:4]
    extra = sys.argv[4:]
    agg, unit = launches(lpath)
    tot = sum(v[1] for v in agg.values())
    lines = [f"# {tag}: ncu launch list (`--metrics gpu__time_duration.sum --clock-control none`)",
             "", "Cold-cache, serialised per-launch times: compare SHARES, not absolutes.", "",
             "| kernel | launches | total | share |", "|---|---|---|---|"]
    for k, (n, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{k[:70]}` | {n} | {v:.0f} {unit} | {100 * v / tot:.1f} % |")
    open(os.path.join(PROF, f"{tag}_launches.md"), "w").write("\n".join(lines) + "\n")
    rep = full(rpath)
    nmain = len(rep)
    for e in extra:
        rep += full(e)
    lines = [f"# {tag}: `ncu --set full` key metrics", ""]
    traffic = {}
    for i, (name, m) in enumerate(rep):
        lines.append(f"## `{name[:110]}`" + ("" if i < nmain else " (extra report)"))
        for k, (v, u) in m.items():
            lines.append(f"- {k}: {v} {u or ''}")
        lines.append("")
        short = next((s for p, s in SHORT.items() if p in name), None)
        if short and i < nmain and short not in traffic and m["dram__bytes_read.sum"][0]:
            b = to_bytes(m["dram__bytes_read.sum"][0], m["dram__bytes_read.sum"][1]) + \
                to_bytes(m["dram__bytes_write.sum"][0], m["dram__bytes_write.sum"][1])
            traffic[short] = b
    open(os.path.join(PROF, f"{tag}_ncu_full.md"), "w").write("\n".join(lines) + "\n")
    if traffic:
        json.dump({**traffic, "source": f"{tag}: ncu --set full, dram__bytes_read.sum + "
                   "dram__bytes_write.sum per launch"}, open(os.path.join(PROF, "ncu_traffic.json"), "w"),
                  indent=1)
    print(open(os.path.join(PROF, f"{tag}_launches.md")).read())


if __name__ == "__main__":
    main()
