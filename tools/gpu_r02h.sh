# grid barrier cost + ncu of the persistent C4 step kernels
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/gridsync_bench tools/gridsync_bench.cu && ./gpurun_out/gridsync_bench | tee gpurun_out/r02h_gridsync.txt
CMD="python bench.py --config C4 --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --no-epoch --graph off"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"persist_step" -s 2 -c 2 -o gpurun_out/r02h_persist $CMD > gpurun_out/r02h_ncu.log 2>&1; echo ncu_rc=$?
tail -2 gpurun_out/r02h_ncu.log
