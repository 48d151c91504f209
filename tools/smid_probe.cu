#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* out) {
    if (threadIdx.x == 0) { int s; asm volatile("mov.u32 %0, %%smid;" : "=r"(s)); out[blockIdx.x] = s; }
}
int main() {
    int* d; cudaMalloc(&d, 592 * 4);
    extern __shared__ char x[];
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 50000);
    void* args[] = {&d};
    cudaLaunchCooperativeKernel((void*)k, 592, 256, args, 50000, 0);
    int h[592]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("coop 592x256 smem50K: first 24 blocks -> smid:");
    for (int i = 0; i < 24; ++i) printf(" %d", h[i]);
    printf("\nblocks 148..155:"); for (int i = 148; i < 156; ++i) printf(" %d", h[i]);
    printf("\n");
    k<<<125, 256>>>(d); cudaMemcpy(h, d, 125*4, cudaMemcpyDeviceToHost);
    printf("plain 125x256: first 24 -> smid:"); for (int i = 0; i < 24; ++i) printf(" %d", h[i]); printf("\n");
    return 0;
}
