mkdir -p gpurun_out
for c in C4 C3; do
SMLP_LIB=build_ab/ptime/libsparse_mlp.so python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-epoch --graph off > gpurun_out/r02k_$c.json 2> gpurun_out/r02k_$c.err
grep "persist phases" gpurun_out/r02k_$c.err | tail -4
done
