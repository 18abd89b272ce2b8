"""Stall samples per CUDA source line of one kernel in an ncu report:
python scripts/ncu_lines.py REPORT KERNEL_REGEX [launch_skip] [top]"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", f"regex:{kern}",
                      "--launch-skip", skip, "--launch-count", "1"], capture_output=True, text=True).stdout
cur, hdr = None, None
agg, src = collections.Counter(), {}
for r in csv.reader(io.StringIO(out)):
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0].isdigit():
        try:
            s = float(r[4])
        except ValueError:
            continue
        agg[(cur, int(r[0]))] += s
        src[(cur, int(r[0]))] = r[1]
tot = sum(agg.values()) or 1
print(f"total samples {tot:.0f}")
for (f, l), s in agg.most_common(top):
    print(f"{s / tot * 100:5.1f}% {f}:{l} {src[(f, l)][:90]}")
