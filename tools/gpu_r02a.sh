# Round-2 first GPU check: full gpu test suite, smoke, default bench, launch list, sanitizers
TAG=${1:-r02a}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/${TAG}_gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -rs > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo bench_rc=$?
cat gpurun_out/${TAG}_bench.json
bash tools/sanitize.sh
