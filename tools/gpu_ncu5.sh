# ncu (set full + source counters) of the library's layer-3 fwd (chunk 0) and bwd (chunk 3) row kernels
TAG=${1:-ncu}
rm -rf /tmp/ncu; mkdir -p /tmp/ncu
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-epoch"
$CMD > /tmp/ncu/plain.log 2>&1; echo plain_rc=$?
for pair in "lf 1" "lb 13"; do
  set -- $pair
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"^(fwd_rows|bwd_rows)_kernel$" -s $2 -c 1 -o /tmp/ncu/$1 $CMD > /tmp/ncu/$1.txt 2>&1; echo rc=$?
  tail -3 /tmp/ncu/$1.txt
  ncu -i /tmp/ncu/$1.ncu-rep --page raw --csv > gpurun_out/${TAG}_$1.csv 2>/dev/null
  ncu -i /tmp/ncu/$1.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_$1_sass.csv 2>/dev/null
done
python tools/ncu_summary.py gpurun_out/${TAG}_lf.csv gpurun_out/${TAG}_lb.csv
