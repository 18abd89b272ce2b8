cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/map
timeout -s KILL 900 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider -k "config4 or u8 or int8 or full_size or trajectory or paged or golden" 2>&1 | tail -1
timeout -s KILL 600 ncu --profile-from-start off --clock-control none --metrics gpu__time_duration.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,smsp__inst_executed.sum -k regex:swa_attend -s 1 -c 1 --csv python bench.py --config 4 --profile-only --steps 2 --warmup 3 2>/dev/null | grep -v "^==" | tail -4 | cut -c1-50,180-400
bash scripts/ab_libs.sh 4 headmap main
