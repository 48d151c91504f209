// gridsync_bench.cu -- cost of one grid-wide barrier on this GPU (persistent step):
// cooperative_groups grid.sync() vs a hand-rolled sense-reversing barrier (one atomic per block
// on a counter, acquire-spin on a generation word), for 1/2/4 blocks per SM of 256 threads.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gridsync_bench tools/gridsync_bench.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdio>

namespace cg = cooperative_groups;

__global__ void cg_kernel(int iters) {
    cg::grid_group g = cg::this_grid();
    for (int i = 0; i < iters; ++i) g.sync();
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// bar[0] = arrivals, bar[1] = generation
__global__ void my_kernel(int iters, unsigned* bar) {
    const unsigned nb = gridDim.x;
    for (int i = 0; i < iters; ++i) {
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned gen = ld_acquire(bar + 1);
            __threadfence();
            if (atomicAdd(bar, 1u) == nb - 1) {
                bar[0] = 0;
                __threadfence();
                atomicAdd(bar + 1, 1u);
            } else {
                while (ld_acquire(bar + 1) == gen) {
                }
            }
        }
        __syncthreads();
    }
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned* bar;
    cudaMalloc(&bar, 8);
    cudaMemset(bar, 0, 8);
    const int iters = 2000;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int per_sm : {1, 2, 4}) {
        const int grid = per_sm * sms;
        for (int variant = 0; variant < 2; ++variant) {
            float best = 1e9f;
            for (int rep = 0; rep < 5; ++rep) {
                cudaEventRecord(a);
                if (variant == 0) {
                    int it = iters;
                    void* args[] = {&it};
                    cudaLaunchCooperativeKernel((void*)cg_kernel, grid, 256, args, 0, 0);
                } else {
                    int it = iters;
                    void* args[] = {&it, &bar};
                    cudaLaunchCooperativeKernel((void*)my_kernel, grid, 256, args, 0, 0);
                }
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (ms < best) best = ms;
            }
            cudaError_t e = cudaGetLastError();
            printf("%-10s blocks %4d (%d/SM): %.3f us per barrier %s\n", variant ? "atomic-gen" : "cg::grid", grid,
                   per_sm, best * 1e3f / iters, e == cudaSuccess ? "" : cudaGetErrorString(e));
        }
    }
    return 0;
}
