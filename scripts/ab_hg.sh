# head-group A/B: bash scripts/ab_hg.sh CONFIG HG...  (0 = the library's choice)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
c=$1; shift
for rep in 1 2; do for hg in "$@"; do
  if [ "$hg" = "0" ]; then unset SKV_HG; else export SKV_HG=$hg; fi
  timeout -s KILL 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-parity > gpurun_out/hg_${c}_$hg.log 2>&1
  python - <<PY
import json
for l in open("gpurun_out/hg_${c}_$hg.log"):
    if l.startswith("{"):
        d=json.loads(l); r=d["roofline"]
        print("c$c hg=$hg", round(d["value"]), "ms", round(d["ms_per_step"],4), "step", round(r["step_frac"],4), "chain", round(r["frac"],4), "iso", round(r["isolated_frac"],4), r["launch"])
PY
done; done
unset SKV_HG
