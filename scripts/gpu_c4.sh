# INT8 attend iteration: config-4 GPU tests, bench config 4, one ncu capture of the attend
TAG=${1:-c4}
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$TAG
timeout -s KILL 600 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider -k "config4 or u8 or int8 or full_size or trajectory" > gpurun_out/$TAG/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/$TAG/pytest_gpu.log
timeout -s KILL 600 python bench.py --config 4 --steps 30 --warmup 5 > gpurun_out/$TAG/bench_c4.jsonl 2>gpurun_out/$TAG/bench_c4.err; echo "bench c4 rc=$?"
timeout -s KILL 600 ncu --profile-from-start off --clock-control none --set full --import-source on -k regex:swa_attend -s 1 -c 1 \
    -o gpurun_out/$TAG/attend_c4 python bench.py --config 4 --profile-only --steps 2 --warmup 3 > gpurun_out/$TAG/attend_c4.json 2>&1; echo "ncu rc=$?"
