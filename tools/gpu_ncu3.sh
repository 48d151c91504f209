# ncu --set full of layer-3 fwd / bwd chunk-0 launches for each SMLP_KVER given (C5 bench step).
# Keeps only CSV exports (raw + source) so gpurun_out stays small.
TAG=${1:-ncu}; shift
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-epoch"
$CMD > gpurun_out/${TAG}_plain.log 2>&1; echo plain_rc=$?
mkdir -p /tmp/ncu
for kv in "$@"; do
  for sk in 1 13; do
    SMLP_KVER=$kv timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^(fwd_rows|bwd_rows|fwd|bwd)_kernel$" -s $sk -c 1 -o /tmp/ncu/${TAG}_k${kv}_s${sk} $CMD > /tmp/ncu/log_${kv}_${sk}.txt 2>&1; echo ncu_rc=$?
    ncu -i /tmp/ncu/${TAG}_k${kv}_s${sk}.ncu-rep --page raw --csv > gpurun_out/${TAG}_k${kv}_s${sk}_raw.csv 2>/dev/null
    ncu -i /tmp/ncu/${TAG}_k${kv}_s${sk}.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_k${kv}_s${sk}_sass.csv 2>/dev/null
  done
done
ls -la gpurun_out/ | tail
