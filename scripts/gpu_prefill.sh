# usage: bash scripts/gpu_prefill.sh  -- prefill parity tests, then the prefill timing
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_gpu_prefill.py -q -x --timeout 120 -p no:cacheprovider > gpurun_out/pytest_prefill.log 2>&1; rc=$?; echo "prefill rc=$rc"; grep -E "Error|passed|failed" gpurun_out/pytest_prefill.log | tail -8
[ $rc = 0 ] && timeout -s KILL 300 python scripts/prefill_bench.py --iters 10 2>&1 | tail -4
