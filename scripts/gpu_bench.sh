# usage: bash scripts/gpu_bench.sh TAG -- default bench line, reference arm, other configs
TAG=${1:-r1}
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt; lscpu | grep -E "Model name|^CPU\(s\)|Thread|Socket" >> gpurun_out/nproc.txt
timeout -s KILL 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
timeout -s KILL 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?"
for c in 1 3 4; do
  timeout -s KILL 900 python bench.py --config $c --no-cpu-baseline --steps 30 > gpurun_out/bench_c${c}_$TAG.json 2> gpurun_out/bench_c${c}_$TAG.err; echo "config $c rc=$?"
done
cat gpurun_out/bench_$TAG.json gpurun_out/bench_ref_$TAG.json; for c in 1 3 4; do tail -c 1500 gpurun_out/bench_c${c}_$TAG.json; echo; tail -3 gpurun_out/bench_c${c}_$TAG.err; done
