# the bench lines alone (configs 2, 3, 4, 1 + the reference arm) into gpurun_out/OUTDIR
OUT=${1:-finalb}
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$OUT
for c in 2 3 4 1; do
  timeout -s KILL 900 python bench.py --config $c --steps 30 --warmup 5 > gpurun_out/$OUT/bench_c$c.jsonl 2>&1; echo "bench c$c rc=$?"
done
timeout -s KILL 900 python bench.py --impl reference --config 2 --steps 3 --warmup 3 > gpurun_out/$OUT/ref_c2.jsonl 2>&1; echo "ref c2 rc=$?"
