nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/smid_probe tools/smid_probe.cu && ./gpurun_out/smid_probe
