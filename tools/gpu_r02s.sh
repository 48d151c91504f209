#!/bin/bash
# A/B: recompute of the implicit delta with packed FFMA2 (rcf2) against the in-tree library (cur)
mkdir -p gpurun_out
SMLP_LIB=build_ab/rcf2/libsparse_mlp.so timeout 900 python -m pytest tests/test_gpu_paths.py -m gpu -x -q -k "implicit_delta" 2>&1 | tail -3
bash tools/gpu_ab_libs.sh r02s cur rcf2 cur rcf2 | grep -E "==|bwd L4|bwd L3|rc="
