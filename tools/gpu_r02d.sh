# PDL A/B on one box (head = last commit's library, main = PDL, nopdl), radix-select evolve parity,
# bounds-checked build over the small parity cases
mkdir -p gpurun_out
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-epoch"
for rep in 1 2; do
for v in head main nopdl; do
  if [ $v = main ]; then L=""; else L="SMLP_LIB=build_ab/$v/libsparse_mlp.so"; fi
  env $L $B > gpurun_out/r02d_c5_${v}_$rep.json 2>&1; python tools/summarize_bench.py gpurun_out/r02d_c5_${v}_$rep.json 2>/dev/null | head -1
  for c in C4 C3; do env $L $B --config $c > gpurun_out/r02d_${c}_${v}_$rep.json 2>&1; python tools/summarize_bench.py gpurun_out/r02d_${c}_${v}_$rep.json 2>/dev/null | head -1; done
done
done
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -rs -k "evolve or prune or topology or overlapped or nccl or dp_k_ranks or long_rows" > gpurun_out/r02d_pytest.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/r02d_pytest.log
SMLP_LIB=build_ab/bounds/libsparse_mlp.so timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -rs -k "long_rows or fused_steps or forward or binary or parity and not full_size and not curves" > gpurun_out/r02d_bounds_pytest.log 2>&1; echo bounds_pytest_rc=$?
tail -3 gpurun_out/r02d_bounds_pytest.log
