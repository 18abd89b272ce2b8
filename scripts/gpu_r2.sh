# usage: bash scripts/gpu_r2.sh [configs...] -- GPU tests + bench lines (with parity) into gpurun_out/
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests -m gpu -q --timeout 400 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_gpu.log | tail -15
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
for c in ${@:-2}; do
  timeout -s KILL 900 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/bench_c$c.log 2>&1; echo "bench c$c rc=$?"
  python - <<PY
import json
for l in open("gpurun_out/bench_c$c.log"):
    if l.startswith("{"):
        d=json.loads(l); r=d.get("roofline") or {}; pf=d.get("prefill") or {}
        print("c$c", round(d["value"]), "step_frac", r.get("step_frac"), "chain_frac", r.get("frac"), "iso", r.get("isolated_frac"),
              "e2e", (d.get("e2e") or {}).get("value"), "prefill", pf.get("ms_per_layer"), pf.get("tflops"), "parity", d.get("parity"),
              "cpu", (d.get("cpu_baseline") or {}).get("value"), d.get("phases"))
PY
  tail -3 gpurun_out/bench_c$c.log | grep -v '^{' | tail -3
done
