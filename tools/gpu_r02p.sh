#!/bin/bash
# A/B of library variants (build_ab/<v>/): parity suite under the variants named in $PYV, then the
# C5 bench with the per-kernel table under each.  PYV="v1 v2" bash tools/gpu_r02p.sh <tag> <variant>...
TAG=$1; shift
mkdir -p gpurun_out
for v in $PYV; do
  SMLP_LIB=build_ab/$v/libsparse_mlp.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_paths.py tests/test_gpu_persist.py \
      -m gpu -x -q -k "not loss_curve" > gpurun_out/${TAG}_${v}_pytest.log 2>&1; echo "pytest[$v] rc=$?"
  tail -3 gpurun_out/${TAG}_${v}_pytest.log
done
bash tools/gpu_ab_libs.sh $TAG "$@"
