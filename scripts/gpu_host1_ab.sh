# single-layer host-buffer step: caller's stream only (new) vs the copy-stream pipeline (SKV_HOST_STREAMS=1),
# config 1 e2e, twice; then the host-step tests
TAG=${1:-host1ab}
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$TAG
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "host_pipelined or entry_pdl" > gpurun_out/$TAG/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/$TAG/pytest.log
for rep in 1 2; do for v in new streams; do
  if [ $v = streams ]; then E="SKV_HOST_STREAMS=1"; else E="SKV_X=1"; fi
  env $E timeout -s KILL 600 python bench.py --config 1 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/$TAG/b_$v$rep.log 2>&1
  python -c "
import json
for l in open('gpurun_out/$TAG/b_$v$rep.log'):
    if l.startswith('{'):
        d=json.loads(l); print('c1 $v', round(d['value']), 'e2e', round(d['e2e']['value']), 'parity', d['parity'].get('idx_mismatch'))"
done; done
