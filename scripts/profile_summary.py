"""Condense one scripts/profile_round.sh run (gpurun_out/TAG_*) into tracked
evidence: profiles/TAG.md (launch list share, per-config attend capture with
DRAM traffic against the algorithmic bytes, the prefill capture) and
profiles/traffic.json (read by bench.py for roofline.traffic).

    python scripts/profile_summary.py TAG
"""
from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)
from summarize_profiles import KEYS, full, launches  # noqa: E402

import bench  # noqa: E402

EXTRA = ["sm__pipe_tensor_op_tcgen05_cycles_active.avg.pct_of_peak_sustained_active"]


def full_all(rep):
    """Every launch of a capture: [(metrics, kernel name)]."""
    import csv
    import io
    import subprocess

    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    if len(rows) < 3:
        return []
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        res, name = {}, ""
        for i, h in enumerate(hdr):
            if h == "Kernel Name":
                name = vals[i]
            if h in KEYS + EXTRA:
                res[h] = f"{vals[i]} {units[i]}".strip()
        out.append((res, name))
    return out


def num(v):
    try:
        return float(str(v).split()[0].replace(",", ""))
    except (ValueError, IndexError):
        return None


def scaled_bytes(v):
    x, unit = num(v), str(v).split()[-1] if v else ""
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1) if x is not None else None


def bench_line(path):
    for line in open(path):
        if line.startswith("{"):
            return json.loads(line)
    return None


def main():
    tag = sys.argv[1]
    g = lambda name: os.path.join(ROOT, "gpurun_out", f"{tag}_{name}")  # noqa: E731
    md = [f"# ncu evidence `{tag}`", "",
          "Produced by `scripts/profile_round.sh` on one B200 (ncu --profile-from-start off: only the bench's "
          "timed region is seen) and summarised by `scripts/profile_summary.py`. Numbers under ncu are not bench "
          "values; launch times are cold-cache and serialised (no PDL overlap).", ""]
    if os.path.exists(g("launches_c2.csv")):
        agg = launches(g("launches_c2.csv"))
        tot = sum(sum(v) for v in agg.values())
        md += ["## Launch list, config 2 timed region (3 steps x 32 layers)", "",
               "| kernel | launches | mean us | total us | share |", "|---|---|---|---|---|"]
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            md.append(f"| `{k}` | {len(v)} | {sum(v) / len(v):.2f} | {sum(v):.1f} | {sum(v) / tot:.3f} |")
        md.append("")
    traffic = {}
    for c in (2, 3, 4):
        rep = g(f"attend_c{c}.ncu-rep")
        if not os.path.exists(rep):
            continue
        res, name = full(rep)
        line = bench_line(g(f"attend_c{c}.json"))
        n = line["profile_capture"]["n_first"]
        algo = bench.attend_algo_bytes(bench.CONFIGS[c], n)
        rd, wr = scaled_bytes(res.get("dram__bytes_read.sum")), scaled_bytes(res.get("dram__bytes_write.sum"))
        dur_us = num(res.get("gpu__time_duration.sum"))
        dram = (rd or 0) + (wr or 0)
        traffic[str(c)] = {"dram_bytes": dram, "algo_bytes": algo, "n": n, "dram_over_algo": dram / algo,
                           "ncu_duration_us": dur_us, "capture": f"profiles/{tag}.md (ncu --set full, layer 1 of "
                                                                  f"the first timed step, n={n})"}
        md += [f"## Attend, config {c} (`{name.split('(')[0]}`), one launch at n={n}", "",
               f"Algorithmic bytes {algo / 1e6:.2f} MB; DRAM read+write {dram / 1e6:.2f} MB "
               f"(ratio {dram / algo:.3f}); under ncu {dur_us} us = {algo / (dur_us * 1e-6) / 1e9:.0f} GB/s "
               "algorithmic (cold, isolated launch).", "", "| metric | value |", "|---|---|"]
        md += [f"| {k} | {res[k]} |" for k in KEYS if k in res]
        md.append("")
    rep = g("select_c2.ncu-rep")
    if os.path.exists(rep):
        res, name = full(rep)
        md += [f"## Select, config 2 (`{name.split('(')[0]}`): the step's batched fold + selection "
               "(grid = sequences x layers)", "", "| metric | value |", "|---|---|"]
        md += [f"| {k} | {res[k]} |" for k in KEYS if k in res]
        md.append("")
    for fname, (B, H, s, D), shape in (("prefill.ncu-rep", (64, 32, 512, 128), "config-2 shape B=64 H=32 s=512 fp16"),
                                       ("prefill2.ncu-rep", (32, 32, 2048, 128),
                                        "config-5 prompt B=32 H=32 s=2048 fp16 (CTA pairs)")):
        rep = g(fname)
        if not os.path.exists(rep):
            continue
        fl = 4.0 * B * H * (s * (s + 1) / 2) * D
        for res, name in full_all(rep):
            dur_us = num(res.get("gpu__time_duration.sum"))
            md += [f"## Prefill (`{name.split('(')[0]}`), {shape}", "",
                   f"Causal GEMM flops of the layer {fl / 1e9:.1f} GFLOP (the two passes together); this launch "
                   f"{dur_us} us.", "", "| metric | value |", "|---|---|"]
            md += [f"| {k} | {res[k]} |" for k in KEYS + EXTRA if k in res]
            md.append("")
    open(os.path.join(ROOT, "profiles", f"{tag}.md"), "w").write("\n".join(md))
    if traffic:
        json.dump(traffic, open(os.path.join(ROOT, "profiles", "traffic.json"), "w"), indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main()
