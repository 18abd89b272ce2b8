# A/B of an environment switch on one box: bash scripts/ab_env.sh CONFIG "ENV=VAL" ...  ("-" = no switch)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
c=$1; shift
for rep in 1 2; do
for ev in "$@"; do
  if [ "$ev" = "-" ]; then E=""; else E="$ev"; fi
  env $E timeout -s KILL 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-parity > gpurun_out/abenv.log 2>&1
  python - "$ev" <<PY
import json,sys
for l in open("gpurun_out/abenv.log"):
    if l.startswith("{"):
        d=json.loads(l); r=d["roofline"]
        print("c$c", sys.argv[1], round(d["value"]), "ms", round(d["ms_per_step"],4), "step", round(r["step_frac"],4), "chain", round(r["frac"],4), "iso", round(r["isolated_frac"],4))
PY
done; done
