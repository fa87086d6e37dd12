"""Summarise ncu captures into profiles/ (tracked).

usage: python tools/ncu_summary.py <round-tag> [gpurun_out/prof_*.ncu-rep ...] [--launches gpurun_out/launches*.csv]

Writes profiles/ncu_<tag>.md (human) and merges the per-kernel numbers into
profiles/ncu_summary.json (bench.py reads roofline.traffic from it).
"""

from __future__ import annotations

import collections
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmalite_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "sm__cycles_elapsed.avg.per_second",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__average_warp_latency_issue_stalled_barrier",
]
UNIT = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "byte": 1.0}


def raw(rep):
    if rep.endswith(".csv"):  # a `--page raw --csv` export made on the GPU box
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for k in METRICS + ["Kernel Name"]:
            if k in hdr:
                d[k] = (r[hdr.index(k)], units[hdr.index(k)])
        res.append(d)
    return res


def to_bytes(v, u):
    try:
        return float(v.replace(",", "")) * UNIT.get(u, 1.0)
    except ValueError:
        return None


def launches(path):
    rows = list(csv.reader(open(path)))
    # find header
    i = next(k for k, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[i]
    kn, mv, mn, unit = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[i + 1:]:
        if len(r) <= mv or r[mn] != "gpu__time_duration.sum":
            continue
        t = float(r[mv].replace(",", ""))
        scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3}.get(r[unit], 1.0)
        name = re.sub(r"\(.*", "", r[kn])
        agg[name][0] += 1
        agg[name][1] += t * scale
    total = sum(v[1] for v in agg.values())
    return total, sorted(agg.items(), key=lambda kv: -kv[1][1])


def main():
    tag = sys.argv[1]
    args = sys.argv[2:sys.argv.index("--launches")] if "--launches" in sys.argv else sys.argv[2:]
    reps = [a for a in args if a.endswith(".ncu-rep") or a.endswith(".csv")]
    lcs = []
    if "--launches" in sys.argv:
        lcs = sys.argv[sys.argv.index("--launches") + 1:]
        lcs = [x for x in lcs if x.endswith(".csv")]
    summ_path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    summ = json.load(open(summ_path)) if os.path.exists(summ_path) else {}
    md = [f"# ncu summary ({tag})", ""]
    for rep in reps:
        m = re.search(r"prof_(\w+?)_(\d+)k?", os.path.basename(rep))
        for d in raw(rep):
            name = d.get("Kernel Name", ("?", ""))[0]
            md.append(f"## {os.path.basename(rep)}: `{name[:90]}`")
            md.append("")
            md.append("| metric | value | unit |")
            md.append("|---|---|---|")
            for k in METRICS:
                if k in d:
                    md.append(f"| {k} | {d[k][0]} | {d[k][1]} |")
            md.append("")
            rd = to_bytes(*d["dram__bytes_read.sum"]) if "dram__bytes_read.sum" in d else None
            wr = to_bytes(*d["dram__bytes_write.sum"]) if "dram__bytes_write.sum" in d else None
            wl = re.sub(r"_r\d+\w*$", "", os.path.basename(rep).replace("prof_", "").replace("raw_", "")
                        .replace(".ncu-rep", "").replace(".csv", ""))
            key = wl  # bench.py workload name
            summ[key] = {
                "kernel": name,
                "dram_bytes": (rd + wr) if rd is not None and wr is not None else None,
                "duration_ms": float(d["gpu__time_duration.sum"][0]) * (1e-3 if d["gpu__time_duration.sum"][1] == "usecond" else 1.0),
                "alu_pipe_pct": float(d["sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"][0]),
                "fma_pipe_pct": float(d["sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"][0]),
                "issue_active_pct": float(d["smsp__issue_active.avg.pct_of_peak_sustained_active"][0]),
                "dram_pct": float(d["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"][0]),
                "warp_instructions": float(d["smsp__inst_executed.sum"][0].replace(",", "")),
                "source": f"{os.path.basename(rep)} ({tag})",
            }
    for lc in lcs:
        total, agg = launches(lc)
        md.append(f"## launch list `{os.path.basename(lc)}` (cold-cache, serialised; compare shares)")
        md.append("")
        md.append("| kernel | launches | total ms | share |")
        md.append("|---|---|---|---|")
        for name, (cnt, ms) in agg:
            md.append(f"| `{name[:80]}` | {cnt} | {ms:.3f} | {ms / total:.1%} |")
        md.append("")
    with open(os.path.join(ROOT, "profiles", f"ncu_{tag}.md"), "w") as f:
        f.write("\n".join(md) + "\n")
    with open(summ_path, "w") as f:
        json.dump(summ, f, indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main()
