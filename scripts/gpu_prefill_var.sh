# usage: bash scripts/gpu_prefill_var.sh VARIANT... -- prefill timings for build_var/lib<variant>.so builds
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python scripts/prefill_bench.py --iters 10 --no-flash 2>&1 | head -1 | sed 's/^/base /'
for v in "$@"; do SKV_LIB=build_var/lib$v.so python scripts/prefill_bench.py --iters 10 --no-flash 2>&1 | head -1 | sed "s/^/$v /"; done
