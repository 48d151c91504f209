# halves + PDL + DP graph: targeted parity, then C5 A/B (halves on/off; PDL on/off), C3/C4 PDL A/B
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -rs -k "long_rows or dp or fused_steps or c5_full_size_sampled" -s > gpurun_out/r02c_pytest.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed|kept per layer" gpurun_out/r02c_pytest.log | tail -5
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-epoch"
$B > gpurun_out/r02c_c5_halves.json 2>gpurun_out/r02c_c5_halves.err; echo rc=$?
python tools/summarize_bench.py gpurun_out/r02c_c5_halves.json
SMLP_BWD_HALF_MIN_BYTES=1000000000000 $B > gpurun_out/r02c_c5_nohalves.json 2>&1; echo rc=$?
python tools/summarize_bench.py gpurun_out/r02c_c5_nohalves.json
SMLP_LIB=build_ab/nopdl/libsparse_mlp.so $B > gpurun_out/r02c_c5_nopdl.json 2>&1; echo rc=$?
python tools/summarize_bench.py gpurun_out/r02c_c5_nopdl.json | head -1
for c in C1 C2 C3 C4; do
  $B --config $c > gpurun_out/r02c_${c}.json 2>&1; python tools/summarize_bench.py gpurun_out/r02c_${c}.json | head -1
  SMLP_LIB=build_ab/nopdl/libsparse_mlp.so $B --config $c > gpurun_out/r02c_${c}_nopdl.json 2>&1; python tools/summarize_bench.py gpurun_out/r02c_${c}_nopdl.json | head -1
  SMLP_BENCH_DP=1 $B --config $c > gpurun_out/r02c_${c}_dp.json 2>&1; python tools/summarize_bench.py gpurun_out/r02c_${c}_dp.json | head -1
done
SMLP_BENCH_DP=1 $B > gpurun_out/r02c_c5_dp.json 2>&1; python tools/summarize_bench.py gpurun_out/r02c_c5_dp.json | head -1
