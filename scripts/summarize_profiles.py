"""Condense ncu outputs from gpurun_out/ into small tracked summaries in profiles/.

    python scripts/summarize_profiles.py TAG [--launches gpurun_out/launches_X.csv]
                                             [--rep gpurun_out/prof_X.ncu-rep] [--note "..."]

Writes profiles/<TAG>.md: the launch list aggregated per kernel (count, mean,
share of GPU time; cold-cache and serialised as ncu replays them) and the key
counters of one `--set full` capture (duration, DRAM bytes and throughput, SM
throughput, occupancy limits, instructions).
"""
from __future__ import annotations

import argparse
import collections
import csv
import io
import os
import subprocess

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__bytes_read.sum.per_second", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_shared_mem",
    "launch__occupancy_limit_registers", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, out = None, collections.defaultdict(list)
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}.get(
                    d["Metric Unit"], 1.0)
                out[d["Kernel Name"].split("(")[0]].append(float(d["Metric Value"].replace(",", "")) * scale)
    return out


def full(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    if len(rows) < 3:
        return {}, ""
    hdr, units = rows[0], rows[1]
    res = {}
    name = ""
    for vals in rows[2:3]:
        for i, h in enumerate(hdr):
            if h == "Kernel Name":
                name = vals[i]
            if h in KEYS:
                res[h] = f"{vals[i]} {units[i]}".strip()
    return res, name


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("tag")
    ap.add_argument("--launches")
    ap.add_argument("--rep")
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    lines = [f"# ncu summary `{a.tag}`", ""]
    if a.note:
        lines += [a.note, ""]
    if a.launches and os.path.exists(a.launches):
        agg = launches(a.launches)
        tot = sum(sum(v) for v in agg.values())
        lines += [f"## Launch list (`{os.path.basename(a.launches)}`: ncu --metrics gpu__time_duration.sum "
                  "--clock-control none; cold-cache, serialised)", "",
                  "| kernel | launches | mean us | total us | share |", "|---|---|---|---|---|"]
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            lines.append(f"| `{k}` | {len(v)} | {sum(v) / len(v):.2f} | {sum(v):.1f} | {sum(v) / tot:.3f} |")
        lines.append("")
    if a.rep and os.path.exists(a.rep):
        res, name = full(a.rep)
        lines += [f"## Full capture (`{os.path.basename(a.rep)}`: ncu --set full, one launch)", "",
                  f"kernel: `{name}`", "", "| metric | value |", "|---|---|"]
        for k in KEYS:
            if k in res:
                lines.append(f"| {k} | {res[k]} |")
        lines.append("")
    os.makedirs("profiles", exist_ok=True)
    out = os.path.join("profiles", f"{a.tag}.md")
    open(out, "w").write("\n".join(lines))
    print(out)


if __name__ == "__main__":
    main()
