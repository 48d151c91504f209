# ncu --set full of one kernel (regex) in a given config's bench step; raw CSV + summary.
# usage: bash tools/gpu_ncu_cfg.sh <tag> <config> <kernel-regex> [skip] [count]
TAG=$1; CFG=$2; K=$3; S=${4:-4}; C=${5:-2}
CMD="python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-epoch --graph off"
$CMD > /tmp/${TAG}_plain.log 2>&1; echo plain_rc=$?
rm -rf /tmp/ncu; mkdir -p /tmp/ncu
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"$K" -s $S -c $C -o /tmp/ncu/k $CMD > /tmp/${TAG}_ncu.log 2>&1; echo ncu_rc=$?
tail -3 /tmp/${TAG}_ncu.log
ncu -i /tmp/ncu/k.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/${TAG}_raw.csv
