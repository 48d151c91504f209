# Full GPU parity suite (no -x: every failure is reported) + smoke.  usage: bash tools/gpu_tests.sh <tag>
TAG=${1:-t}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -rs --durations=15 > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -25 gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo smoke_rc=$?
tail -2 gpurun_out/${TAG}_smoke.log
