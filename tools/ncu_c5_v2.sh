CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-epoch"
$CMD > gpurun_out/plain_v2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5_v2.csv $CMD > gpurun_out/ncu_launch_v2.log 2>&1 ; \
ncu --set full --clock-control none --import-source on -k regex:"fwd_kernel|bwd_kernel" -s 32 -c 32 -o gpurun_out/prof_c5_v2 $CMD > gpurun_out/ncu_full_v2.log 2>&1; echo ncu_rc=$?; tail -2 gpurun_out/ncu_full_v2.log
