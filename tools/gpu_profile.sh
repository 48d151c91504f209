# Round-end evidence on one B200 (each ncu pass only after the same command exited 0 without ncu):
#   1. bench.py default (C5)                            -> gpurun_out/${TAG}_bench.json
#   2. ncu launch list (gpu__time_duration, 1 step)     -> gpurun_out/${TAG}_launches.csv
#   3. ncu --set full of the dominant kernel's launches  -> gpurun_out/${TAG}_dom_raw.csv (+ SASS source page)
TAG=${1:-prof}
DOM=${2:-bwd_rows_kernel}
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-epoch"
timeout 1200 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo bench_rc=$?
$CMD > /tmp/${TAG}_plain.log 2>&1; echo plain_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > /tmp/${TAG}_ncu1.log 2>&1; echo ncu_list_rc=$?
rm -rf /tmp/ncu; mkdir -p /tmp/ncu
# the dominant kernel: all launches of the last (timed) step = the last 2 x (hidden layers) launches
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"^${DOM}$" -s 12 -c 6 -o /tmp/ncu/dom $CMD > /tmp/${TAG}_ncu2.log 2>&1; echo ncu_full_rc=$?
ncu -i /tmp/ncu/dom.ncu-rep --page raw --csv > gpurun_out/${TAG}_dom_raw.csv 2>/dev/null
ncu -i /tmp/ncu/dom.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_dom_sass.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/${TAG}_dom_raw.csv
