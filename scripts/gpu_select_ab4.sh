# incremental select on the fold's long path: the selection tests, then config 4 with / without it (twice)
TAG=${1:-selab4}
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$TAG
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 600 -p no:cacheprovider -k "incremental or trajectory or long" > gpurun_out/$TAG/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/$TAG/pytest.log
for rep in 1 2; do for ev in "-" "SKV_SELECT_FULL=1"; do
  if [ "$ev" = "-" ]; then E=""; else E="$ev"; fi
  env $E timeout -s KILL 600 python bench.py --config 4 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/$TAG/b.log 2>&1
  python -c "
import json
for l in open('gpurun_out/$TAG/b.log'):
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']; par=d.get('parity') or {}
        print('c4', '$ev', round(d['value']), 'ms', round(d['ms_per_step'],4), 'step', round(r['step_frac'],4), 'idx_mismatch', par.get('idx_mismatch'), 'err', round(par.get('max_err_over_tol',0),3))"
done; done
