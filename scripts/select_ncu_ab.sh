# select kernel duration (ncu, timed region only) with the incremental selection and with SKV_SELECT_FULL=1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/selncu
for c in 4 2; do for ev in "-" "SKV_SELECT_FULL=1"; do
  if [ "$ev" = "-" ]; then E=""; T=incr; else E="$ev"; T=full; fi
  env $E timeout -s KILL 600 ncu --profile-from-start off --clock-control none --metrics gpu__time_duration.sum -k regex:swa_select --csv python bench.py --config $c --profile-only --steps 2 --warmup 3 > gpurun_out/selncu/c${c}_$T.csv 2>&1
  python -c "
import csv,io
v=[float(r[-1]) for r in csv.reader(io.StringIO(open('gpurun_out/selncu/c${c}_$T.csv').read())) if len(r)>12 and r[-3]=='gpu__time_duration.sum']
print('c$c', '$T', len(v), 'launches, mean us', round(sum(v)/max(1,len(v))/1000,2))"
done; done
