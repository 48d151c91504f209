#!/bin/bash
# last refresh of the default bench line after the rotate-based sign nibble in the recompute kernel
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_paths.py -m gpu -x -q -k "implicit_delta or c5_full_size_sampled" > gpurun_out/final3_pytest.log 2>&1; echo "pytest rc=$?" | tee -a gpurun_out/final3_pytest.log
tail -3 gpurun_out/final3_pytest.log
python bench.py > gpurun_out/final3_bench_c5.json 2> gpurun_out/final3_bench_c5.err; echo "bench rc=$?"
python tools/summarize_bench.py gpurun_out/final3_bench_c5.json
python bench.py --config T1 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-epoch > gpurun_out/final3_bench_T1.json 2> gpurun_out/final3_bench_T1.err; python tools/summarize_bench.py gpurun_out/final3_bench_T1.json | head -1
python bench.py --config T2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-epoch > gpurun_out/final3_bench_T2.json 2> gpurun_out/final3_bench_T2.err; python tools/summarize_bench.py gpurun_out/final3_bench_T2.json | head -1
