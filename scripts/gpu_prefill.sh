cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_prefill.py -q -x --timeout 200 -p no:cacheprovider > gpurun_out/pytest_prefill.log 2>&1; echo "prefill rc=$?"; tail -25 gpurun_out/pytest_prefill.log
timeout -s KILL 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -8 gpurun_out/pytest_gpu.log
