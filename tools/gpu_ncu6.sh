# ncu (set full + SASS source counters) of one launch of the kernel named $2 in a C5 bench step
TAG=${1:-ncu}; K=$2; SKIP=${3:-0}
rm -rf /tmp/ncu; mkdir -p /tmp/ncu
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-epoch"
$CMD > /tmp/ncu/plain.log 2>&1; echo plain_rc=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"^${K}$" -s $SKIP -c 1 -o /tmp/ncu/k $CMD > /tmp/ncu/k.txt 2>&1; echo rc=$?
tail -2 /tmp/ncu/k.txt
ncu -i /tmp/ncu/k.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>/dev/null
ncu -i /tmp/ncu/k.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_sass.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/${TAG}_raw.csv
