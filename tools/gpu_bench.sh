# C5 bench only (kernel timings), one line summary per env setting
TAG=${1:-b}; shift
n=0
for envs in "$@"; do
  n=$((n+1))
  env $envs timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-epoch $BENCH_ARGS > gpurun_out/${TAG}_c5_$n.json 2> gpurun_out/${TAG}_c5_$n.err; echo "bench[$envs]_rc=$?"
  python tools/summarize_bench.py gpurun_out/${TAG}_c5_$n.json
done
