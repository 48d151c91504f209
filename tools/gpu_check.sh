# One GPU round: parity tests, smoke, default bench (with cpu_baseline / e2e / epoch),
# then the ncu launch list and one --set full capture of the fwd/bwd kernels of one C5 step.
# usage (from the repo root, under gpurun): bash tools/gpu_check.sh <tag>
TAG=${1:-run}
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/${TAG}_gpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo pytest_rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo bench_rc=$?
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-epoch"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launch.log 2>&1 ; echo ncu1_rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"${NCU_REGEX:-fwd_kernel|bwd_kernel}" -s ${NCU_SKIP:-32} -c ${NCU_COUNT:-32} -o gpurun_out/${TAG}_prof $CMD > gpurun_out/${TAG}_ncu_full.log 2>&1; echo ncu2_rc=$?
tail -3 gpurun_out/${TAG}_ncu_full.log
