# launch list (ncu per-kernel durations) of the timed region of one config: bash scripts/gpu_launches.sh TAG CONFIG [sel]
TAG=${1:-ll}; C=${2:-4}
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$TAG
timeout -s KILL 600 ncu --profile-from-start off --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  --log-file gpurun_out/$TAG/launches_c$C.csv python bench.py --config $C --profile-only --steps 2 --warmup 3 > gpurun_out/$TAG/launches_c$C.json 2>&1; echo "launches rc=$?"
if [ -n "$3" ]; then
timeout -s KILL 600 ncu --profile-from-start off --clock-control none --set full --import-source on -k regex:swa_select -s 1 -c 1 \
    -o gpurun_out/$TAG/select_c$C python bench.py --config $C --profile-only --steps 2 --warmup 3 > /dev/null 2>&1; echo "select ncu rc=$?"
fi
