# compute-sanitizer over the decode parity tests after the config-1 attend changes (entry-wait PDL, the
# warp-shared softmax, the 8-stage fp32 ring): memcheck over the trajectories, racecheck + synccheck over
# the single-layer fp32 / bf16 paths (the ones the shared-memory softmax exchange runs in)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/san_r2h
CS=/usr/local/cuda/bin/compute-sanitizer
K="decode_trajectory or golden_trajectory or decode_ratios or decode_from_first or attend_over_indices or multilayer_step"
timeout -s KILL 1500 $CS --tool memcheck --leak-check no --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "$K and not config4_full" > gpurun_out/san_r2h/memcheck_decode.log 2>&1; echo "memcheck rc=$?"; tail -3 gpurun_out/san_r2h/memcheck_decode.log
timeout -s KILL 1500 $CS --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "golden_trajectory or decode_from_first or (decode_trajectory and f32)" > gpurun_out/san_r2h/racecheck_decode.log 2>&1; echo "racecheck rc=$?"; tail -3 gpurun_out/san_r2h/racecheck_decode.log
timeout -s KILL 1500 $CS --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "golden_trajectory or decode_from_first or (decode_trajectory and f32)" > gpurun_out/san_r2h/synccheck_decode.log 2>&1; echo "synccheck rc=$?"; tail -3 gpurun_out/san_r2h/synccheck_decode.log
