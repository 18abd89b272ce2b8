# usage: bash scripts/gpu_prefill_perf.sh  -- prefill timings + ncu launch list of the config-2 shape
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout -s KILL 600 python scripts/prefill_bench.py --iters 10 2>&1 | tee gpurun_out/prefill_bench.log | tail -5
cat > /tmp/pf_one.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
from paper_2403_17312_b200 import api
B, H, s, D = 64, 32, 512, 128
k = torch.randn(B, s, H, D, device="cuda").half(); v = torch.randn_like(k); q = torch.randn_like(k) * 0.5
c = api.SwaCache(1, B, H, D, s, kv_dtype="f16"); c.append_tokens(0, 0, 0, k, v)
for _ in range(3): c.prefill_layer(0, q)
torch.cuda.synchronize()
PY
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/prefill_launches.csv python /tmp/pf_one.py > gpurun_out/prefill_ncu.log 2>&1; echo "ncu rc=$?"
