mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_persist.py -q -x --timeout 600 -rs > gpurun_out/r02o_persist.log 2>&1; echo persist_rc=$?
tail -3 gpurun_out/r02o_persist.log
B="python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e --no-epoch"
for c in C1 C2 C3 C4; do
  $B --config $c > gpurun_out/r02o_${c}.json 2>&1; python tools/summarize_bench.py gpurun_out/r02o_${c}.json
  SMLP_PERSIST=0 $B --config $c > gpurun_out/r02o_${c}_k.json 2>&1; python tools/summarize_bench.py gpurun_out/r02o_${c}_k.json | head -1
done
for c in C4 C3; do
SMLP_LIB=build_ab/ptime/libsparse_mlp.so python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-epoch --graph off > gpurun_out/r02o_t$c.json 2> gpurun_out/r02o_t$c.err
grep "persist phases" gpurun_out/r02o_t$c.err | tail -2
done
