#!/bin/bash
# compute-sanitizer over the library's kernels (only kernels in the smlp namespace are checked;
# torch's own kernels are excluded).  Logs: gpurun_out/sanitize_<tool>.log
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "memcheck" ] && extra="--leak-check no"
  timeout 1800 /usr/local/cuda/bin/compute-sanitizer --tool $tool $extra --kernel-name regex:smlp \
      --print-limit 50 python tools/sanitize_workload.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "== $tool rc=$?: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize_$tool.log | tail -1)"
done
