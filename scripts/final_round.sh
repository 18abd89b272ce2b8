# end-of-round evidence on one box: GPU tests, smoke, bench configs 1-5 (+ parity), reference arm, the ncu
# round, prefill timing beside flash_attn / cuDNN, config-1 / config-4 step anatomy, MMA cost probe.
# usage: bash scripts/final_round.sh OUTDIR NCU_TAG   (outputs under gpurun_out/OUTDIR, gpurun_out/NCU_TAG_*)
OUT=${1:-final}; TAG=${2:-r2}
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$OUT
timeout -s KILL 1500 python -m pytest tests -m gpu -q -rs --timeout 600 -p no:cacheprovider > gpurun_out/$OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/$OUT/pytest_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/$OUT/smoke.log 2>&1; echo "smoke rc=$?"
for c in 2 3 4 1; do
  timeout -s KILL 900 python bench.py --config $c --steps 30 --warmup 5 > gpurun_out/$OUT/bench_c$c.jsonl 2>&1; echo "bench c$c rc=$?"
done
timeout -s KILL 900 python bench.py --impl reference --config 2 --steps 3 --warmup 3 > gpurun_out/$OUT/ref_c2.jsonl 2>&1; echo "ref c2 rc=$?"
timeout -s KILL 1800 python bench.py --config 5 > gpurun_out/$OUT/bench_c5.jsonl 2>&1; echo "bench c5 rc=$?"
timeout -s KILL 600 python scripts/prefill_bench.py > gpurun_out/$OUT/prefill_bench.jsonl 2>&1; echo "prefill bench rc=$?"
timeout -s KILL 300 python scripts/c1_probe.py > gpurun_out/$OUT/c1_probe.log 2>&1; echo "c1 probe rc=$?"
PF=1 KV2=1 ROT=1 TRACE=1 timeout -s KILL 600 python scripts/step_probe.py > gpurun_out/$OUT/c4_step_probe.log 2>&1; echo "c4 probe rc=$?"
[ -x build_var/mma_probe ] && timeout -s KILL 120 ./build_var/mma_probe > gpurun_out/$OUT/mma_probe.log 2>&1; echo "mma probe rc=$?"
# NO_NCU=1: skip the ncu round (its .ncu-rep files can push gpurun_out past the 64 MiB copy-back limit)
[ -z "$NO_NCU" ] && { bash scripts/profile_round.sh $TAG > gpurun_out/$OUT/profile_round.log 2>&1; echo "profile rc=$?"; }
