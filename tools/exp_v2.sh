timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 2>&1 | tail -15
for cb in 0 128 64 16; do
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-epoch --chunk-batch $cb > gpurun_out/bench_c5_v2_cb$cb.json 2>&1
done
python bench.py --config C2 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --no-epoch > gpurun_out/bench_c2_v2.json 2>&1
