# select change check: all GPU tests, the parity soak, then configs 2 / 3 / 1 with the incremental select vs SKV_SELECT_FULL=1 (twice)
TAG=${1:-selab}
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$TAG
timeout -s KILL 1500 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/$TAG/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/$TAG/pytest_gpu.log
timeout -s KILL 900 python scripts/parity_soak.py --seeds 12 > gpurun_out/$TAG/soak.log 2>&1; echo "soak rc=$?"; tail -2 gpurun_out/$TAG/soak.log
for rep in 1 2; do for c in 2 3 1; do for ev in "-" "SKV_SELECT_FULL=1"; do
  if [ "$ev" = "-" ]; then E=""; else E="$ev"; fi
  env $E timeout -s KILL 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/$TAG/b.log 2>&1
  python -c "
import json,sys
for l in open('gpurun_out/$TAG/b.log'):
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']; par=d.get('parity') or {}
        print('c$c', '$ev', round(d['value']), 'ms', round(d['ms_per_step'],4), 'step', round(r['step_frac'],4), 'idx_mismatch', par.get('idx_mismatch'), 'err', round(par.get('max_err_over_tol',0),3))"
done; done; done
