cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_prefill.py -q --timeout 200 -p no:cacheprovider > gpurun_out/pytest_prefill.log 2>&1; echo "prefill rc=$?"; grep -E "Error|passed|failed" gpurun_out/pytest_prefill.log | tail -12
timeout -s KILL 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
