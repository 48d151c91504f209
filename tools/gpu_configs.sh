# bench.py on every config (kernel timings only), one summary line each
for c in C1 C2 C3 C4; do
  timeout 600 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --no-epoch > gpurun_out/cfg_$c.json 2> gpurun_out/cfg_$c.err; echo "$c rc=$?"
  python -c "
import json; d=json.loads(open('gpurun_out/cfg_$c.json').read().strip().splitlines()[-1])
print('$c', d['value'], 'samples/s', d['ms_per_step'], 'ms/step', 'F1 frac', d['step_roofline']['frac'], 'CB', d['config']['chunk_batch'], 'launches', d['gpu_launches'])"
done
