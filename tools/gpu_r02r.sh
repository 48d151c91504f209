#!/bin/bash
# implicit delta_{L-1}: parity (new test), then the C5 bench with the records path off / on
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_paths.py -m gpu -x -q -k "implicit_delta" > gpurun_out/r02r_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r02r_pytest.log
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-epoch"
for rep in 1 2; do
  SMLP_IMPLICIT_DELTA=0 $B > gpurun_out/r02r_off.json 2> gpurun_out/r02r_off.err; echo "off rc=$?"; python tools/summarize_bench.py gpurun_out/r02r_off.json | grep -E "==|bwd L"
  $B > gpurun_out/r02r_on.json 2> gpurun_out/r02r_on.err; echo "on rc=$?"; python tools/summarize_bench.py gpurun_out/r02r_on.json | grep -E "==|bwd L"
done
