# A/B the ring configuration variants in variants/*.so on configs 2,3,4
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
summ() { python -c "
import json,sys
d=json.loads(open('$1').read().strip().splitlines()[-1]); r=d['roofline']
print(round(d['value']), 'tok/s | kernel', round(r['frac'],3), round(r['kernel_ms_avg']*1000,1), 'us | step', round(r['step_frac'],3))" 2>&1 | tail -1; }
for lib in default variants/lib_b8k6.so variants/lib_b8k4.so variants/lib_b16k3.so variants/lib_b16k2.so; do
  for c in 2 3 4; do
    if [ $lib = default ]; then unset SKV_LIB; else export SKV_LIB=$GRAFT_REPO_ROOT/$lib; fi
    timeout -s KILL 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/var.log 2>&1
    echo "$lib c$c: $(summ gpurun_out/var.log)"
  done
done
