# round-2 batch: GPU tests, head-shard exchange overhead (config 3), config 5 full
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests -m gpu -q --timeout 400 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_gpu.log | tail -8
timeout -s KILL 600 python bench.py --config 3 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-parity > gpurun_out/c3_plain.log 2>&1; echo "c3 plain rc=$?"
timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --config 3 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-parity --shard-exchange > gpurun_out/c3_exchange.log 2>&1; echo "c3 exchange rc=$?"
for f in c3_plain c3_exchange; do python - <<PY
import json
for l in open("gpurun_out/$f.log"):
    if l.startswith("{"):
        d=json.loads(l); r=d["roofline"]; print("$f", round(d["value"]), "ms", round(d["ms_per_step"],4), "step_frac", round(r["step_frac"],4), d["config"]["parallelism"])
PY
done
if [ "${C5:-1}" = "1" ]; then timeout -s KILL 1500 python bench.py --config 5 > gpurun_out/bench_c5_full.log 2>&1; echo "c5 rc=$?"; fi
