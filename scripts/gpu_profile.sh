# usage: bash scripts/gpu_profile.sh TAG [full]  -- tests, HG sweep, ncu launch list (+ full capture)
TAG=${1:-r1}
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
for hg in 0 2 4 8; do
  SKV_HG=$hg timeout -s KILL 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_hg$hg.log 2>&1
  echo "HG=$hg $(python -c "
import json
d=json.loads(open('gpurun_out/bench_hg$hg.log').read().strip().splitlines()[-1]); r=d['roofline']
print(round(d['value']), 'tok/s', round(d['ms_per_step'],3), 'ms/step | kernel', round(r['achieved']), 'GB/s', round(r['kernel_ms_avg']*1000,1), 'us | step', round(r['step_achieved']), 'GB/s', round(r['step_frac'],3))" 2>&1 | tail -1)"
done
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --profile-only --steps 3 --warmup 3 > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
if [ "$2" = "full" ]; then
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:swa_attend -s 70 -c 1 -o gpurun_out/prof_$TAG python bench.py --profile-only --steps 2 --warmup 3 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
tail -2 gpurun_out/ncu_full.log
fi
