# ncu (set full, CSV only) of: library fwd/bwd row kernels (layer 3, chunk 0) and the microbench row kernel
TAG=${1:-ncu}
rm -rf /tmp/ncu; mkdir -p /tmp/ncu
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-epoch"
$CMD > /tmp/ncu/plain.log 2>&1; echo plain_rc=$?
[ -z "$SKIP_LIB" ] && timeout 600 ncu --set full --clock-control none -k regex:"^(fwd_rows|bwd_rows)_kernel$" -s 1 -c 1 -o /tmp/ncu/lf $CMD > /tmp/ncu/l1.txt 2>&1; echo rc=$?
[ -z "$SKIP_LIB" ] && timeout 600 ncu --set full --clock-control none -k regex:"^(fwd_rows|bwd_rows)_kernel$" -s 13 -c 1 -o /tmp/ncu/lb $CMD > /tmp/ncu/l2.txt 2>&1; echo rc=$?
ONLY_ROW=1 timeout 600 ncu --set full --clock-control none -k regex:"k_row" -c 1 -o /tmp/ncu/mb ./tools/spmm_bench > /tmp/ncu/m.txt 2>&1; echo rc=$?
for f in lf lb mb; do ncu -i /tmp/ncu/$f.ncu-rep --page raw --csv > gpurun_out/${TAG}_$f.csv 2>/dev/null; done
python tools/ncu_summary.py gpurun_out/${TAG}_lf.csv gpurun_out/${TAG}_lb.csv gpurun_out/${TAG}_mb.csv
