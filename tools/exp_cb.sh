set -x
./tools/gather_bench > gpurun_out/gather_bench.csv 2>&1
for cb in 32 64 16; do
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-epoch --chunk-batch $cb > gpurun_out/bench_c5_cb$cb.json 2>&1
done
