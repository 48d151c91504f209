#!/bin/bash
# A/B: fwd_bits predicated adds (pred) and forward reduce-scatter epilogue (frs = pred + rs)
mkdir -p gpurun_out
for v in frs; do
  SMLP_LIB=build_ab/$v/libsparse_mlp.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_paths.py -m gpu -x -q \
      -k "binary or forward or chunk or long_rows or c5_full_size_sampled or fused_steps" > gpurun_out/r02q_${v}_pytest.log 2>&1; echo "pytest[$v] rc=$?"
  tail -3 gpurun_out/r02q_${v}_pytest.log
done
bash tools/gpu_ab_libs.sh r02q base pred frs base pred frs
