# Iteration run on one B200: GPU parity tests, then the C5 / C2 benches (kernel timings only).
# usage (repo root, under gpurun): bash tools/gpu_iter.sh <tag> [pytest -k expr]
TAG=${1:-iter}
K=${2:-}
set -x
if [ -n "$K" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -k "$K" > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo pytest_rc=$?
else
  timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo pytest_rc=$?
fi
tail -30 gpurun_out/${TAG}_pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-epoch > gpurun_out/${TAG}_bench_c5.json 2> gpurun_out/${TAG}_bench_c5.err; echo bench_rc=$?
timeout 300 python bench.py --config C2 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --no-epoch > gpurun_out/${TAG}_bench_c2.json 2> gpurun_out/${TAG}_bench_c2.err; echo bench2_rc=$?
python tools/summarize_bench.py gpurun_out/${TAG}_bench_c5.json gpurun_out/${TAG}_bench_c2.json
