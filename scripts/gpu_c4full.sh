# one ncu --set full capture of the config-4 attend (INT8) + summary lines
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/c4full
timeout -s KILL 600 ncu --profile-from-start off --clock-control none --set full --import-source on -k regex:swa_attend -s 1 -c 1 \
  -o gpurun_out/c4full/attend_c4 python bench.py --config 4 --profile-only --steps 2 --warmup 3 > gpurun_out/c4full/attend_c4.json 2>&1; echo "ncu rc=$?"
timeout -s KILL 600 python bench.py --config 4 --steps 30 --warmup 5 > gpurun_out/c4full/bench_c4.jsonl 2>/dev/null; echo "bench rc=$?"
