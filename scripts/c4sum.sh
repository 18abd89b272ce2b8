# summarize a config-4 iteration: bash scripts/c4sum.sh TAG
T=$1
python -c "
import json
d=json.loads(open('gpurun_out/$T/bench_c4.jsonl').read().strip().splitlines()[-1]); r=d['roofline']
print('c4', round(d['value']), round(d['ms_per_step'],4), 'frac',round(r['frac'],3),'step',round(r['step_frac'],3),'iso',round(r['isolated_frac'],3), 'e2e', round(d['e2e']['value']), 'parity', round(d['parity']['max_err_over_tol'],3), d['parity']['idx_mismatch'], d['clocks']['sm_mhz'], d['clocks']['reasons'])
"
ncu -i gpurun_out/$T/attend_c4.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,smsp__inst_executed.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,launch__registers_per_thread 2>/dev/null | python -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h=rows[0]
print({k.split('.')[0].replace('l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op','conf'):v for k,v in zip(h,rows[2]) if any(x in k for x in ['duration','dram','inst_exec','conflicts','throughput','registers'])})
"
