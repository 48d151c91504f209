#!/bin/bash
# Round-2 final bench + ncu evidence with the in-tree library (the whole GPU suite ran in
# tools/gpu_r02_final.sh; here the tests that touch the kernels changed since)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_paths.py tests/test_gpu_parity.py -m gpu -x -q -k "implicit_delta or c5_full_size_sampled or fused_steps or chunked" > gpurun_out/final2_pytest.log 2>&1; echo "pytest rc=$?" | tee -a gpurun_out/final2_pytest.log
tail -3 gpurun_out/final2_pytest.log
python bench.py > gpurun_out/final2_bench_c5.json 2> gpurun_out/final2_bench_c5.err; echo "bench rc=$?"
python tools/summarize_bench.py gpurun_out/final2_bench_c5.json
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-epoch"
$CMD > /dev/null 2>&1; echo "plain rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/final2_ncu_launches_c5.csv $CMD > gpurun_out/final2_ncu_launches.log 2>&1; echo "ncu list rc=$?"
python tools/launch_share.py gpurun_out/final2_ncu_launches_c5.csv > gpurun_out/final2_ncu_launch_share_c5.txt; cat gpurun_out/final2_ncu_launch_share_c5.txt
rm -rf /tmp/ncu; mkdir -p /tmp/ncu
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"bwd_rows|fwd_rows" -s 30 -c 12 -o /tmp/ncu/k $CMD > /tmp/ncu/k.txt 2>&1; echo "ncu full rc=$?"
ncu -i /tmp/ncu/k.ncu-rep --page raw --csv > gpurun_out/final2_ncu_rows_raw.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/final2_ncu_rows_raw.csv > gpurun_out/final2_ncu_rows_summary.txt; cat gpurun_out/final2_ncu_rows_summary.txt
