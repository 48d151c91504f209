# C5 chunk-width sweep: bench per (CB:CBf) spec
for spec in "$@"; do
  IFS=: read -r cb cbf <<< "$spec"
  SMLP_FWD_CB=$cbf timeout 600 python bench.py --chunk-batch $cb --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-epoch > gpurun_out/c5sw_${cb}_${cbf}.json 2> gpurun_out/c5sw_${cb}_${cbf}.err
  echo "[$spec] rc=$?"; python tools/summarize_bench.py gpurun_out/c5sw_${cb}_${cbf}.json 2>/dev/null | head -1
done
