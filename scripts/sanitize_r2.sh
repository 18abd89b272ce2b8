# compute-sanitizer memcheck over the round-2 GPU paths (paged store, ledger, engine, boundary)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout -s KILL 2400 $CS --tool memcheck --leak-check no --print-limit 20 python -m pytest tests/test_gpu_paged.py tests/test_gpu_ledger.py -q -p no:cacheprovider -k "not int8" > gpurun_out/memcheck_paged.log 2>&1; echo "memcheck paged rc=$?"; tail -3 gpurun_out/memcheck_paged.log
timeout -s KILL 1200 $CS --tool memcheck --leak-check no --print-limit 20 tests/cpp/build/engine_parity > gpurun_out/memcheck_engine.log 2>&1; echo "memcheck engine rc=$?"; tail -3 gpurun_out/memcheck_engine.log
timeout -s KILL 1200 $CS --tool memcheck --leak-check no --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "dense_attention or unsorted or errors" > gpurun_out/memcheck_boundary.log 2>&1; echo "memcheck boundary rc=$?"; tail -3 gpurun_out/memcheck_boundary.log
