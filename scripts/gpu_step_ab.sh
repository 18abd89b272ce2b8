# whole-step change check: all GPU tests + the parity soak on the new build, then configs 2 / 4 / 3 with the
# new build vs build_var/libbase.so (the previous commit), twice
TAG=${1:-c1ab}
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$TAG
timeout -s KILL 1500 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/$TAG/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/$TAG/pytest_gpu.log
timeout -s KILL 900 python scripts/parity_soak.py --seeds 6 > gpurun_out/$TAG/soak.log 2>&1; echo "soak rc=$?"; tail -1 gpurun_out/$TAG/soak.log
for rep in 1 2; do for lib in new base; do
  if [ $lib = base ]; then E="SKV_LIB=build_var/libbase.so"; else E="SKV_X=1"; fi
  for c in 2 4 3; do
  env $E timeout -s KILL 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/$TAG/b.log 2>&1
  python -c "
import json,sys
for l in open('gpurun_out/$TAG/b.log'):
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']; par=d.get('parity') or {}
        print('c$c', '$lib', round(d['value']), 'ms', round(d['ms_per_step'],4), 'step', round(r['step_frac'],4), 'idx_mismatch', par.get('idx_mismatch'), 'err', round(par.get('max_err_over_tol',0),3))"
  done
done; done
