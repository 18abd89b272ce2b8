# usage: bash scripts/gpu_prefill_var.sh VARIANT... -- interleaved prefill timings of build_var/lib<variant>.so builds
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2; do for v in "$@"; do SKV_LIB=build_var/lib$v.so timeout -s KILL 120 python scripts/prefill_bench.py --iters 10 --no-flash 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l); print('$v', d['shape'][:8], d['ms'])
    except Exception: pass
"; done; done
