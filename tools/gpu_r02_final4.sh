#!/bin/bash
# end of round 2: the whole GPU suite and the default bench line with the final in-tree library
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/final4_pytest_gpu.log 2>&1; echo "pytest rc=$?" | tee -a gpurun_out/final4_pytest_gpu.log
tail -3 gpurun_out/final4_pytest_gpu.log
python bench.py > gpurun_out/final4_bench_c5.json 2> gpurun_out/final4_bench_c5.err; echo "bench rc=$?"
python tools/summarize_bench.py gpurun_out/final4_bench_c5.json
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-epoch"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/final4_ncu_launches_c5.csv $CMD > gpurun_out/final4_ncu_launches.log 2>&1; echo "ncu list rc=$?"
python tools/launch_share.py gpurun_out/final4_ncu_launches_c5.csv > gpurun_out/final4_ncu_launch_share_c5.txt; cat gpurun_out/final4_ncu_launch_share_c5.txt
python __graft_entry__.py smoke 2>&1 | tail -2
