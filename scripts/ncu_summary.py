"""Summarise an ncu --set full report: per kernel duration, throughput, occupancy
and the top warp-stall reasons, plus the hottest SASS lines.
    python scripts/ncu_summary.py REPORT.ncu-rep [--sass N]"""
import csv
import io
import subprocess
import sys


def ncu(args):
    return subprocess.run(["ncu", "-i", sys.argv[1]] + args, capture_output=True, text=True).stdout


def main():
    nsass = int(sys.argv[sys.argv.index("--sass") + 1]) if "--sass" in sys.argv else 0
    rows = list(csv.reader(io.StringIO(ncu(["--page", "raw", "--csv"]))))
    hdr = rows[0]
    want = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_tensor_op_tcgen05_cycles_active.avg.pct_of_peak_sustained_active" ,
            "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
            "launch__occupancy_limit_shared_mem"]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        print(d["Kernel Name"][:70])
        for k in want:
            for kk in d:
                if kk == k:
                    print(f"   {k:70s} {d[kk]}")
        st = []
        for k, v in d.items():
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                try:
                    st.append((float(v.replace(",", "")), k[len("smsp__pcsamp_warps_issue_stalled_"):]))
                except ValueError:
                    pass
        tot = sum(v for v, _ in st) or 1
        print("   stalls:", ", ".join(f"{n} {v / tot:.0%}" for v, n in sorted(st, reverse=True)[:7]))
    if nsass:
        text = ncu(["--page", "source", "--csv", "--print-source", "sass"])
        blocks, cur = [], None
        for ln in text.split("\n"):
            if ln.startswith('"Kernel Name"'):
                cur = [ln]
                blocks.append(cur)
            elif cur is not None:
                cur.append(ln)
        for b in blocks:
            rr = list(csv.reader(b[1:]))
            h = rr[0]
            data = [dict(zip(h, x)) for x in rr[1:] if len(x) == len(h)]
            print(b[0][:100])
            for d in sorted(data, key=lambda d: -int(d["Warp Stall Sampling (All Samples)"]))[:nsass]:
                print(f'   {d["Warp Stall Sampling (All Samples)"]:>6} {d["Address"][-5:]} {d["Source"][:80]}')


if __name__ == "__main__":
    main()
