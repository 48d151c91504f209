# round-2 measurement pass: gather ceiling (2nd roofline), default bench line, DP-path graphs,
# ncu launch list + one full capture of the C5 hidden-layer fwd / bwd row kernels
mkdir -p gpurun_out
timeout 600 python tools/gather_ceiling.py --out gpurun_out/gather_ceiling.json > gpurun_out/r02e_ceiling.log 2>&1; echo ceiling_rc=$?
mkdir -p profiles && cp gpurun_out/gather_ceiling.json profiles/gather_ceiling.json 2>/dev/null
timeout 1200 python bench.py > gpurun_out/r02e_bench.json 2> gpurun_out/r02e_bench.err; echo bench_rc=$?
python tools/summarize_bench.py gpurun_out/r02e_bench.json | head -3
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-epoch"
for c in C4 C3; do $B --config $c > gpurun_out/r02e_${c}.json 2>&1; python tools/summarize_bench.py gpurun_out/r02e_${c}.json | head -1
  SMLP_BENCH_DP=1 $B --config $c > gpurun_out/r02e_${c}_dp.json 2>&1; python tools/summarize_bench.py gpurun_out/r02e_${c}_dp.json | head -1; done
SMLP_BENCH_DP=1 $B > gpurun_out/r02e_c5_dp.json 2>&1; python tools/summarize_bench.py gpurun_out/r02e_c5_dp.json | head -1
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-epoch --graph off"
$CMD > gpurun_out/r02e_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02e_launches.csv $CMD > gpurun_out/r02e_ncu_launch.log 2>&1 ; echo ncu1_rc=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"bwd_rows_kernel|fwd_rows_kernel" -s 12 -c 4 -o gpurun_out/r02e_prof $CMD > gpurun_out/r02e_ncu_full.log 2>&1; echo ncu2_rc=$?
tail -2 gpurun_out/r02e_ncu_full.log
