# round-2 final evidence on one box: GPU tests, smoke, bench configs 1-4 (+ parity), config 5 full, ncu round
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/final
timeout -s KILL 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/final/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/final/pytest_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo "smoke rc=$?"
for c in 2 3 4 1; do
  timeout -s KILL 900 python bench.py --config $c --steps 30 --warmup 5 > gpurun_out/final/bench_c$c.jsonl 2>&1; echo "bench c$c rc=$?"
done
timeout -s KILL 900 python bench.py --impl reference --config 2 --steps 3 --warmup 3 > gpurun_out/final/ref_c2.jsonl 2>&1; echo "ref c2 rc=$?"
timeout -s KILL 1800 python bench.py --config 5 > gpurun_out/final/bench_c5.jsonl 2>&1; echo "bench c5 rc=$?"
bash scripts/profile_round.sh r2 > gpurun_out/final/profile_round.log 2>&1; echo "profile rc=$?"
