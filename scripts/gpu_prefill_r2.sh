# prefill evidence: timing vs flash_attn / cuDNN SDPA, and one ncu --set full capture of each pass (config-2 shape)
TAG=${1:-pf}
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$TAG
timeout -s KILL 600 python scripts/prefill_bench.py > gpurun_out/$TAG/prefill_bench.jsonl 2>gpurun_out/$TAG/prefill_bench.err; echo "bench rc=$?"; cat gpurun_out/$TAG/prefill_bench.jsonl
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:flash_prefill -s 2 -c 2 \
  -o gpurun_out/$TAG/prefill python scripts/prefill_one.py > gpurun_out/$TAG/prefill_ncu.log 2>&1; echo "ncu rc=$?"
