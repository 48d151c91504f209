# A/B run on one B200: GPU parity tests, then the C5 bench under each env setting given.
# usage: bash tools/gpu_ab.sh <tag> "ENV=.. ENV2=.." "ENV=.." ...   (first arg after tag = A, ...)
TAG=${1:-ab}; shift
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/${TAG}_pytest_gpu.log
n=0
for envs in "$@"; do
  n=$((n+1))
  env $envs timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-epoch > gpurun_out/${TAG}_c5_$n.json 2> gpurun_out/${TAG}_c5_$n.err; echo "bench[$envs]_rc=$?"
  python tools/summarize_bench.py gpurun_out/${TAG}_c5_$n.json
done
