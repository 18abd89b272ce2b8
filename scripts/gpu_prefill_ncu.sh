# usage: bash scripts/gpu_prefill_ncu.sh TAG -- launch list + full capture of both flash passes
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; TAG=${1:-pf}
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python scripts/prefill_one.py > /dev/null 2>&1; echo "list rc=$?"
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:flash_prefill -s 2 -c 2 -o gpurun_out/${TAG}_full python scripts/prefill_one.py > gpurun_out/${TAG}_ncu.log 2>&1; echo "full rc=$?"; tail -2 gpurun_out/${TAG}_ncu.log
