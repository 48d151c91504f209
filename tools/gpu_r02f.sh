# small configs: ncu launch list (kernel durations) of eager steps vs the graph-replayed step time
mkdir -p gpurun_out
for c in C4 C3 C1; do
  CMD="python bench.py --config $c --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --no-epoch --graph off"
  $CMD > gpurun_out/r02f_${c}_plain.json 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02f_${c}_launches.csv $CMD > gpurun_out/r02f_${c}_ncu.log 2>&1; echo ncu_${c}_rc=$?
  python tools/launch_share.py gpurun_out/r02f_${c}_launches.csv 2>&1 | head -30
done
