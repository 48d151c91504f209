# A/B of library env settings on the C5 bench (kernel timings), then optional pytest selection.
# usage: PYTEST_K="expr" bash tools/gpu_ab_env.sh <tag> "ENV=a" "ENV=b" ...
TAG=${1:-ab}; shift
mkdir -p gpurun_out
if [ -n "$PYTEST_K" ]; then
  timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -rs -k "$PYTEST_K" > gpurun_out/${TAG}_pytest.log 2>&1; echo pytest_rc=$?
  tail -5 gpurun_out/${TAG}_pytest.log
fi
n=0
for envs in "$@"; do
  n=$((n+1))
  env $envs timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-epoch $BENCH_ARGS > gpurun_out/${TAG}_$n.json 2> gpurun_out/${TAG}_$n.err; echo "bench[$envs]_rc=$?"
  python tools/summarize_bench.py gpurun_out/${TAG}_$n.json
done
