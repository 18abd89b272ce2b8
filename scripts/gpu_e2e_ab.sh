# e2e (host-buffer) leg of configs 3 / 2: current build, SKV_SELECT_FULL=1, and the build before incremental selection
TAG=${1:-e2eab}
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$TAG
for rep in 1 2; do for c in 3 2; do for v in new full preincr; do
  case $v in new) E="SKV_X=1";; full) E="SKV_SELECT_FULL=1";; preincr) E="SKV_LIB=build_var/libpreincr.so";; esac
  env $E timeout -s KILL 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-parity > gpurun_out/$TAG/b_${c}_${v}_$rep.log 2>&1
  python -c "
import json
for l in open('gpurun_out/$TAG/b_${c}_${v}_$rep.log'):
    if l.startswith('{'):
        d=json.loads(l); print('c$c $v', round(d['value']), 'e2e', round(d['e2e']['value']), 'enq', d.get('host_enqueue_ms_per_step'))"
done; done; done
