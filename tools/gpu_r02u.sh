#!/bin/bash
# A/B: Eq. 1 + mirror refresh of W^(3..L) on the side stream under the bit kernels of W^(2) (early)
mkdir -p gpurun_out
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-epoch"
for rep in 1 2; do
for v in cur early; do
  SMLP_LIB=build_ab/$v/libsparse_mlp.so $B > gpurun_out/r02u_$v.json 2> gpurun_out/r02u_$v.err; echo "bench[$v] rc=$?"
  python tools/summarize_bench.py gpurun_out/r02u_$v.json | grep -E "==|bwd_bits|sgd_update|layer_update"
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/r02u_$v.json') if l.startswith('{')][-1]); print('   e2e', round(d['e2e']['value'],1), 'profiled', d.get('ms_per_step_profiled'))"
done; done
SMLP_LIB=build_ab/early/libsparse_mlp.so timeout 1200 python -m pytest tests/test_gpu_paths.py -m gpu -x -q -k "c5_full_size_sampled or pipelined_host_step" 2>&1 | tail -3
