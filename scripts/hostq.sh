cd $GRAFT_REPO_ROOT
for c in 4 2 1; do timeout -s KILL 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-parity 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
  if l.startswith('{'): d=json.loads(l); print('c$c', round(d['ms_per_step'],4), 'host', round(d['host_enqueue_ms_per_step'],4), 'step', round(d['roofline']['step_frac'],3), 'chain', round(d['roofline']['frac'],3))
"; done
