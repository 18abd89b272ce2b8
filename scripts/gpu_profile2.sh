TAG=${1:-r1v3}
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout -s KILL 300 python scripts/gemm_bench.py > gpurun_out/gemm_bench.json 2>&1; cat gpurun_out/gemm_bench.json
# launch list of 2 decode steps (skip prompt setup: 32 writes + 32 seed attends + 32 seed selects)
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"swa_|ledger|kv_move|gemm|recompute" -s 96 -c 200 --csv --log-file gpurun_out/launches_c2_$TAG.csv python bench.py --profile-only --steps 3 --warmup 3 > /dev/null 2>&1; echo "c2 launches rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:swa_attend -s 70 -c 1 -o gpurun_out/prof_c2_$TAG python bench.py --profile-only --steps 2 --warmup 3 > /dev/null 2>&1; echo "c2 full rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:swa_attend -s 200 -c 1 -o gpurun_out/prof_c4_$TAG python bench.py --config 4 --profile-only --steps 2 --warmup 3 > /dev/null 2>&1; echo "c4 full rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tn -s 2 -c 1 -o gpurun_out/prof_gemm_$TAG python scripts/gemm_bench.py > /dev/null 2>&1; echo "gemm full rc=$?"
