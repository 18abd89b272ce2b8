# quick iteration on one box: GPU tests, bench configs given as args, one attend capture of config 4
# usage: bash scripts/gpu_iter.sh TAG "4 2" [ncu-configs]
TAG=${1:-it}; CFGS=${2:-"4"}; NCFG=${3:-"4"}
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$TAG
timeout -s KILL 900 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/$TAG/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/$TAG/pytest_gpu.log
for c in $CFGS; do
  timeout -s KILL 600 python bench.py --config $c --steps 30 --warmup 5 > gpurun_out/$TAG/bench_c$c.jsonl 2>gpurun_out/$TAG/bench_c$c.err; echo "bench c$c rc=$?"
done
for c in $NCFG; do
  timeout -s KILL 600 ncu --profile-from-start off --clock-control none --set full --import-source on -k regex:swa_attend -s 1 -c 1 \
    -o gpurun_out/$TAG/attend_c$c python bench.py --config $c --profile-only --steps 2 --warmup 3 > gpurun_out/$TAG/attend_c$c.json 2>&1
  echo "ncu c$c rc=$?"
done
