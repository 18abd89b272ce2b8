# compute-sanitizer memcheck + racecheck-free check of the prefill tests (1-CTA and CTA-pair kernels) on the final code,
# then the parity soak (seeded oracle trajectories)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/san_final
CS=/usr/local/cuda/bin/compute-sanitizer
timeout -s KILL 1800 $CS --tool memcheck --leak-check no --print-limit 20 python -m pytest tests/test_gpu_prefill.py -q -p no:cacheprovider -k "not both_kernels" > gpurun_out/san_final/memcheck_prefill.log 2>&1; echo "memcheck prefill rc=$?"; tail -3 gpurun_out/san_final/memcheck_prefill.log
timeout -s KILL 1800 python scripts/parity_soak.py --seeds 24 > gpurun_out/san_final/parity_soak.log 2>&1; echo "soak rc=$?"; tail -5 gpurun_out/san_final/parity_soak.log
