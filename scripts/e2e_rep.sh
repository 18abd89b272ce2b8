cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/e2erep
for c in 2 3 2 3 2; do
  timeout -s KILL 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-parity > gpurun_out/e2erep/b.log 2>&1
  python - $c <<'P'
import json,sys
for l in open("gpurun_out/e2erep/b.log"):
    if l.startswith("{"):
        d=json.loads(l); print("c"+sys.argv[1], round(d["value"]), "e2e", round(d["e2e"]["value"]), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
P
done
