# persistent step: bitwise A/B tests, the small-config GPU suite on the persistent path, benches
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_persist.py -q -x --timeout 600 -rs > gpurun_out/r02g_persist.log 2>&1; echo persist_rc=$?
tail -30 gpurun_out/r02g_persist.log | head -60
B="python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e --no-epoch"
for c in C1 C2 C3 C4; do
  $B --config $c > gpurun_out/r02g_${c}.json 2>&1; python tools/summarize_bench.py gpurun_out/r02g_${c}.json | head -1
  SMLP_PERSIST=0 $B --config $c > gpurun_out/r02g_${c}_k.json 2>&1; python tools/summarize_bench.py gpurun_out/r02g_${c}_k.json | head -1
done
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -rs -k "not full_size" > gpurun_out/r02g_pytest.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/r02g_pytest.log
