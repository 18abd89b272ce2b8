# ncu full capture of the attend kernel (+ a select kernel) for configs 3 and 4
TAG=${1:-r1}
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in 3 4; do
  L=$([ $c = 3 ] && echo 40 || echo 48)
  timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:swa_attend -s $((L+L*3)) -c 1 -o gpurun_out/prof_c${c}_$TAG python bench.py --config $c --profile-only --steps 2 --warmup 3 > gpurun_out/ncu_c$c.log 2>&1; echo "ncu c$c rc=$?"
  timeout -s KILL 900 ncu --set full --clock-control none -k regex:swa_select -s $((L+L*3)) -c 1 -o gpurun_out/prof_sel_c${c}_$TAG python bench.py --config $c --profile-only --steps 2 --warmup 3 > gpurun_out/ncu_sel_c$c.log 2>&1; echo "ncu sel c$c rc=$?"
done
