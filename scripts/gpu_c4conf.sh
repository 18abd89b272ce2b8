# INT8 / decode shared-memory conflict check: GPU decode tests, one ncu conflict count per config, A/B vs build_var/lib$1.so
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider -k "config4 or u8 or int8 or full_size or trajectory or paged or golden or variants or long or host" 2>&1 | tail -1
for c in 4 2 1; do
timeout -s KILL 600 ncu --profile-from-start off --clock-control none --metrics gpu__time_duration.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum -k regex:swa_attend -s 1 -c 1 --csv python bench.py --config $c --profile-only --steps 2 --warmup 3 2>/dev/null | grep -v "^==" | tail -3 | cut -c1-40,180-400
done
[ -n "$1" ] && bash scripts/ab_libs.sh 4 $1 main && bash scripts/ab_libs.sh 2 $1 main
