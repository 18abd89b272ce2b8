cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/mr
export BENCH_DIST_BACKEND=gloo BENCH_DEVICE=0
for c in 2 1; do
timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/mr/c$c.log 2>&1; echo "c$c rc=$?"; grep '^{' gpurun_out/mr/c$c.log | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['n_gpus'], d['scaling'], round(d['value']), d['config'].get('parallelism'), d.get('e2e',{}) and round(d['e2e']['value']), (d.get('parity') or {}).get('idx_mismatch'))"
done
timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > gpurun_out/mr/ref.log 2>&1; echo "ref rc=$?"; grep -c '^{' gpurun_out/mr/ref.log
