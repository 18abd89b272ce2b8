# prefill change check: the prefill GPU tests, then prefill_bench.py (no flash_attn) twice
TAG=${1:-pfab}
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$TAG
timeout -s KILL 900 python -m pytest tests/test_gpu_prefill.py -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/$TAG/pytest_prefill.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/$TAG/pytest_prefill.log
for rep in 1 2; do
  timeout -s KILL 300 python scripts/prefill_bench.py --no-flash > gpurun_out/$TAG/bench_$rep.jsonl 2>&1; echo "bench rc=$?"
  python -c "
import json,sys
for l in open('gpurun_out/$TAG/bench_$rep.jsonl'):
    if l.startswith('{'): d=json.loads(l); print(d['shape'], d['ms'], 'cudnn', d.get('cudnn_sdpa_ms'))"
done
