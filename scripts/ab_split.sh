# A/B of the side-stream select split: bash scripts/ab_split.sh [configs]
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in ${@:-4 2 3}; do
  for sp in 0 -1; do
    if [ "$sp" = "-1" ]; then unset SKV_SELECT_SPLIT; else export SKV_SELECT_SPLIT=$sp; fi
    timeout -s KILL 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-parity > gpurun_out/ab_c${c}_s${sp}.log 2>&1
    python - <<PY
import json
for l in open("gpurun_out/ab_c${c}_s${sp}.log"):
    if l.startswith("{"):
        d=json.loads(l); r=d["roofline"]
        print("c$c split=$sp", round(d["value"]), "ms", round(d["ms_per_step"],4), "step_frac", round(r["step_frac"],4), "chain", round(r["frac"],4))
PY
  done
done
unset SKV_SELECT_SPLIT
