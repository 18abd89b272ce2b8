# usage: bash scripts/profile_round.sh TAG -- ncu evidence for profiles/:
#  launch list of the default bench's timed region (cold-cache, serialised),
#  one --set full attend capture per config (layer 1 of the first timed step;
#  the bench JSON line beside it gives that step's n), the prefill passes.
TAG=${1:-r1}
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
NCU="ncu --profile-from-start off --clock-control none"
timeout -s KILL 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  --log-file gpurun_out/${TAG}_launches_c2.csv python bench.py --profile-only --steps 3 --warmup 3 \
  > gpurun_out/${TAG}_launches_c2.json 2>&1; echo "launch list rc=$?"
for c in 2 3 4; do
  timeout -s KILL 900 $NCU --set full --import-source on -k regex:swa_attend -s 1 -c 1 -o gpurun_out/${TAG}_attend_c$c \
    python bench.py --config $c --profile-only --steps 2 --warmup 3 > gpurun_out/${TAG}_attend_c$c.json 2>&1
  echo "attend c$c rc=$?"
done
timeout -s KILL 900 $NCU --set full -k regex:swa_select -s 1 -c 1 -o gpurun_out/${TAG}_select_c2 \
  python bench.py --config 2 --profile-only --steps 2 --warmup 3 > /dev/null 2>&1; echo "select c2 rc=$?"
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:flash_prefill -s 2 -c 2 \
  -o gpurun_out/${TAG}_prefill python scripts/prefill_one.py > gpurun_out/${TAG}_prefill.log 2>&1; echo "prefill rc=$?"
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:flash2_prefill -s 2 -c 2 \
  -o gpurun_out/${TAG}_prefill2 python scripts/prefill_one.py --c5 > gpurun_out/${TAG}_prefill2.log 2>&1; echo "prefill2 rc=$?"
