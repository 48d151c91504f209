#!/bin/bash
# A/B: delta_{l-1} stores of the recompute kernel with evict_last (e1); rotate-based nibble (e2)
mkdir -p gpurun_out
for v in e1 e2; do SMLP_LIB=build_ab/$v/libsparse_mlp.so timeout 900 python -m pytest tests/test_gpu_paths.py -m gpu -x -q -k "implicit_delta" 2>&1 | tail -1; done
bash tools/gpu_ab_libs.sh r02t cur e1 e2 cur e1 e2 | grep -E "==|bwd L4|bwd L3|rc="
