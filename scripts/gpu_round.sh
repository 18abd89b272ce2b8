# usage: bash scripts/gpu_round.sh -- GPU tests, smoke, bench configs 2/3/4/5 (short), kept in gpurun_out/
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
for c in 2 3 4 5; do
  timeout -s KILL 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c$c.log 2>&1; echo "bench c$c rc=$?"
  python - <<PY
import json
for l in open("gpurun_out/bench_c$c.log"):
    if l.startswith("{"):
        d=json.loads(l); r=d.get("roofline") or {}; pf=d.get("prefill") or {}
        print("c$c", round(d["value"]), d["unit"], "step_frac", r.get("step_frac"), "chain_frac", r.get("frac"),
              "e2e", (d.get("e2e") or {}).get("value"), "prefill", pf.get("ms_per_layer"), pf.get("tflops"), d.get("phases"))
PY
done
