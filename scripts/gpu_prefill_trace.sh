cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
SKV_LIB=build_var/libtrace.so timeout 120 python scripts/prefill_one.py > gpurun_out/trace.log 2>&1; echo rc=$?; wc -l gpurun_out/trace.log
