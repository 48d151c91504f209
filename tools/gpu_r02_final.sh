#!/bin/bash
# Round-2 final measurements with the in-tree library: the whole GPU suite, the default bench (C5),
# the ncu launch list of the same command, a full ncu capture of the two backward row kernels, and
# the small configs.  Everything lands in gpurun_out/final_*.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/final_pytest_gpu.log 2>&1; echo "pytest rc=$?" | tee -a gpurun_out/final_pytest_gpu.log
tail -3 gpurun_out/final_pytest_gpu.log
python bench.py > gpurun_out/final_bench_c5.json 2> gpurun_out/final_bench_c5.err; echo "bench rc=$?"
python tools/summarize_bench.py gpurun_out/final_bench_c5.json
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-epoch"
$CMD > /dev/null 2>&1; echo "plain rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_ncu_launches_c5.csv $CMD > gpurun_out/final_ncu_launches.log 2>&1; echo "ncu list rc=$?"
python tools/launch_share.py gpurun_out/final_ncu_launches_c5.csv > gpurun_out/final_ncu_launch_share_c5.txt; cat gpurun_out/final_ncu_launch_share_c5.txt
rm -rf /tmp/ncu; mkdir -p /tmp/ncu
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"bwd_rows" -s 8 -c 6 -o /tmp/ncu/k $CMD > /tmp/ncu/k.txt 2>&1; echo "ncu full rc=$?"
ncu -i /tmp/ncu/k.ncu-rep --page raw --csv > gpurun_out/final_ncu_bwd_rows_raw.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/final_ncu_bwd_rows_raw.csv > gpurun_out/final_ncu_bwd_rows_summary.txt; cat gpurun_out/final_ncu_bwd_rows_summary.txt
B="python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e --no-epoch"
for c in C1 C2 C3 C4; do
  $B --config $c > gpurun_out/final_bench_${c}.json 2> gpurun_out/final_bench_${c}.err; python tools/summarize_bench.py gpurun_out/final_bench_${c}.json | head -1
done
