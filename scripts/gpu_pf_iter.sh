# prefill iteration: prefill GPU tests, timing vs cuDNN, ncu capture of both passes
TAG=${1:-pf}
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$TAG
timeout -s KILL 600 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider -k "prefill or smoke or headshard" > gpurun_out/$TAG/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/$TAG/pytest_gpu.log
bash scripts/gpu_prefill_r2.sh $TAG
