mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_persist.py -q -x --timeout 600 -rs > gpurun_out/r02j_persist.log 2>&1; echo persist_rc=$?
tail -3 gpurun_out/r02j_persist.log
B="python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e --no-epoch"
for c in C1 C2 C3 C4; do
  $B --config $c > gpurun_out/r02j_${c}.json 2>&1; python tools/summarize_bench.py gpurun_out/r02j_${c}.json
  SMLP_PERSIST=0 $B --config $c > gpurun_out/r02j_${c}_k.json 2>&1; python tools/summarize_bench.py gpurun_out/r02j_${c}_k.json | head -1
done
CMD="python bench.py --config C4 --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --no-epoch --graph off"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"persist_step" -s 2 -c 2 -o gpurun_out/r02j_persist $CMD > gpurun_out/r02j_ncu.log 2>&1; echo ncu_rc=$?
