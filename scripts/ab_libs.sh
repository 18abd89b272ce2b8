# A/B of library builds on one box: bash scripts/ab_libs.sh CONFIG lib1 lib2 ... (build_var/libNAME.so; "main" = the in-tree build)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
c=$1; shift
for rep in 1 2; do
for name in "$@"; do
  if [ "$name" = "main" ]; then unset SKV_LIB; else export SKV_LIB=$GRAFT_REPO_ROOT/build_var/lib$name.so; fi
  timeout -s KILL 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-parity > gpurun_out/ab_${c}_$name.log 2>&1
  python - <<PY
import json
for l in open("gpurun_out/ab_${c}_$name.log"):
    if l.startswith("{"):
        d=json.loads(l); r=d["roofline"]
        print("c$c $name", round(d["value"]), "ms", round(d["ms_per_step"],4), "step", round(r["step_frac"],4), "chain", round(r["frac"],4), "iso", round(r["isolated_frac"],4))
PY
done; done
unset SKV_LIB
