cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in 2 3 4; do for hg in 1 2 4 8; do
  SKV_HG=$hg timeout -s KILL 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/hg.log 2>&1 || { echo "c$c hg$hg failed: $(tail -1 gpurun_out/hg.log)"; continue; }
  python -c "
import json
d=json.loads(open('gpurun_out/hg.log').read().strip().splitlines()[-1]); r=d['roofline']
print('c$c hg$hg', round(d['value']), 'tok/s step', round(r['step_frac'],3), 'chain', round(r['frac'],3), 'iso', round(r['isolated_frac'],3), r['launch'])"
done; done
