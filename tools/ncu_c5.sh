CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-epoch"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv $CMD > gpurun_out/ncu_launch.log 2>&1 ; \
ncu --set full --clock-control none --import-source on -k regex:"fwd_kernel|bwd_kernel" -s 8 -c 8 -o gpurun_out/prof_c5 $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu_rc=$?; tail -3 gpurun_out/ncu_full.log
