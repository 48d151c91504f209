# ncu --set full of selected kernels of one C5 bench step (after the same command ran clean).
# usage: NCU_REGEX='...' NCU_SKIP=n NCU_COUNT=m bash tools/gpu_ncu.sh <tag>
TAG=${1:-ncu}
set -x
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-epoch"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"${NCU_REGEX}" -s ${NCU_SKIP:-0} -c ${NCU_COUNT:-8} -o gpurun_out/${TAG}_prof $CMD > gpurun_out/${TAG}_ncu.log 2>&1; echo ncu_rc=$?
tail -3 gpurun_out/${TAG}_ncu.log
