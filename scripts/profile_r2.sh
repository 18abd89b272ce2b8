# round-2 ncu evidence: launch lists (config 1, 2, 4) + --set full attend captures (config 2, 4)
TAG=${1:-r2}
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
NCU="ncu --profile-from-start off --clock-control none"
for c in 1 2 4; do
  timeout -s KILL 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --csv \
    --log-file gpurun_out/${TAG}_launches_c$c.csv python bench.py --config $c --profile-only --steps 3 --warmup 3 \
    > gpurun_out/${TAG}_launches_c$c.json 2>&1; echo "launch list c$c rc=$?"
done
for c in 2 4; do
  timeout -s KILL 900 $NCU --set full --import-source on -k regex:swa_attend -s 1 -c 1 -o gpurun_out/${TAG}_attend_c$c \
    python bench.py --config $c --profile-only --steps 2 --warmup 3 > gpurun_out/${TAG}_attend_c$c.json 2>&1
  echo "attend c$c rc=$?"
done
timeout -s KILL 900 $NCU --set full -k regex:swa_select -s 1 -c 1 -o gpurun_out/${TAG}_select_c4 \
  python bench.py --config 4 --profile-only --steps 2 --warmup 3 > /dev/null 2>&1; echo "select c4 rc=$?"
