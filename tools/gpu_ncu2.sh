# ncu --set full of the layer-3/4 row kernels of one C5 bench step (fwd: launches 1-2, bwd: 12-13).
TAG=${1:-ncu}
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-epoch"
$CMD > gpurun_out/${TAG}_plain.log 2>&1; echo plain_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^(fwd_rows|bwd_rows)_kernel" -s 1 -c 2 -o gpurun_out/${TAG}_fwd $CMD > gpurun_out/${TAG}_ncu_fwd.log 2>&1; echo ncu_fwd_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^(fwd_rows|bwd_rows)_kernel" -s 12 -c 2 -o gpurun_out/${TAG}_bwd $CMD > gpurun_out/${TAG}_ncu_bwd.log 2>&1; echo ncu_bwd_rc=$?
tail -2 gpurun_out/${TAG}_ncu_fwd.log gpurun_out/${TAG}_ncu_bwd.log
