# Width-scaling sweep (Table 4 rows T1..T5): bench per (config, chunk width[, forward width]).
# usage: bash tools/gpu_width.sh <tag> "T2:32" "T2:64" "T2:128:32" ...   (config:CB[:CBf])
TAG=${1:-w}; shift
for spec in "$@"; do
  IFS=: read -r cfg cb cbf <<< "$spec"
  envs=""; [ -n "$cbf" ] && envs="SMLP_FWD_CB=$cbf"
  out=gpurun_out/${TAG}_${cfg}_${cb}_${cbf:-eq}.json
  env $envs timeout 900 python bench.py --config $cfg --chunk-batch $cb --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-epoch > $out 2> ${out%.json}.err
  echo "bench[$spec]_rc=$?"
  python tools/summarize_bench.py $out | head -1
done
