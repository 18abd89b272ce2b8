# usage: bash scripts/gpu_prefill_list.sh TAG -- ncu launch list of prefill_one.py (f16 and bf16)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; TAG=${1:-pf}
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/${TAG}_list.csv python scripts/prefill_one.py > /dev/null 2>&1; echo "list rc=$?"
python - <<PY
import csv
rows=list(csv.reader(open("gpurun_out/${TAG}_list.csv")))
hdr=None; data={}
for r in rows:
    if r and r[0]=="ID": hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r)); data.setdefault(d["ID"],{"name":d["Kernel Name"][:40]})[d["Metric Name"]]=d["Metric Value"]
for k,v in list(data.items())[-3:]: print(k,v)
PY
