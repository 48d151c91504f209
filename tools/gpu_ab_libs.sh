#!/bin/bash
# C5 bench (per-kernel table) under each A/B library build: bash tools/gpu_ab_libs.sh <tag> <variant>...
# (variants built by tools/ab_build.py into build_ab/<variant>/)
TAG=$1; shift
for v in "$@"; do
  SMLP_LIB=build_ab/$v/libsparse_mlp.so timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-epoch \
      > gpurun_out/${TAG}_$v.json 2> gpurun_out/${TAG}_$v.err; echo "bench[$v] rc=$?"
  python tools/summarize_bench.py gpurun_out/${TAG}_$v.json
done
