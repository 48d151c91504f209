// gather_bench.cu — microbenchmark of random row-gather bandwidth on B200.
//
// The sparse MLP step gathers one B-wide activation / delta row per nonzero per pass; with an
// Erdos-Renyi topology those rows are uniformly random over a slab of n_rows x row_bytes.  This
// measures the achievable gather bandwidth as a function of slab size (L2-resident or not) and
// row size, which is the second ceiling of DESIGN.md ("L2-gather roofline").
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_bench tools/gather_bench.cu
//   ./gather_bench            -> one CSV line per (slab_MB, row_bytes, unroll)
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

template <int ROWB, int U>
__global__ void __launch_bounds__(256) gather_kernel(const float* __restrict__ slab, const int* __restrict__ idx,
                                                     long n_idx, float* __restrict__ out) {
    constexpr int G = ROWB / 16;          // lanes per row (float4 each)
    constexpr int P = 32 / G;             // rows per warp instruction
    const int lane = threadIdx.x & 31, g = lane / G, q = lane % G;
    const long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
    const long nw = (gridDim.x * (long)blockDim.x) >> 5;
    float4 acc = make_float4(0, 0, 0, 0);
    for (long base = warp * 32; base < n_idx; base += nw * 32) {
        const int myidx = idx[base + lane];
#pragma unroll
        for (int t0 = 0; t0 < 32; t0 += P * U) {
            float4 x[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int r = __shfl_sync(0xffffffffu, myidx, (t0 + u * P + g) & 31);
                x[u] = __ldg(reinterpret_cast<const float4*>(slab + (long)r * (ROWB / 4)) + q);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) { acc.x += x[u].x; acc.y += x[u].y; acc.z += x[u].z; acc.w += x[u].w; }
        }
    }
    if (acc.x + acc.y + acc.z + acc.w == 1234.5f) out[0] = acc.x;   // keep the loads alive
}

template <int ROWB, int U>
void run(long slab_bytes, int sms, int blocks_per_sm, float* slab, int* idx, long n_idx, float* out) {
    const long rows = slab_bytes / ROWB;
    std::vector<int> h(n_idx);
    uint64_t s = 88172645463325252ull;
    for (long k = 0; k < n_idx; ++k) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[k] = (int)(s % (uint64_t)rows); }
    CK(cudaMemcpy(idx, h.data(), n_idx * 4, cudaMemcpyHostToDevice));
    const int grid = sms * blocks_per_sm;
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    gather_kernel<ROWB, U><<<grid, 256>>>(slab, idx, n_idx, out);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int it = 0; it < 5; ++it) {
        cudaEventRecord(a);
        gather_kernel<ROWB, U><<<grid, 256>>>(slab, idx, n_idx, out);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    const double bytes = (double)n_idx * ROWB;
    printf("%ld,%d,%d,%d,%.3f,%.1f\n", slab_bytes >> 20, ROWB, U, blocks_per_sm, best, bytes / (best * 1e-3) / 1e9);
    fflush(stdout);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int l2 = 0;
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
    printf("# SMs %d, L2 %d bytes\n", sms, l2);
    printf("slab_MB,row_bytes,unroll,blocks_per_sm,best_ms,gather_GBps\n");
    const long max_slab = 512l << 20;
    const long n_idx = 40l << 20;          // 40M row gathers per launch
    float *slab, *out; int* idx;
    CK(cudaMalloc(&slab, max_slab));
    CK(cudaMemset(slab, 0, max_slab));
    CK(cudaMalloc(&idx, n_idx * 4));
    CK(cudaMalloc(&out, 64));
    for (long mb : {16l, 32l, 64l, 96l, 128l, 256l, 512l}) {
        const long sb = mb << 20;
        run<512, 8>(sb, sms, 4, slab, idx, n_idx / 2, out);
        run<256, 8>(sb, sms, 4, slab, idx, n_idx / 2, out);
        run<128, 8>(sb, sms, 4, slab, idx, n_idx, out);
        run<64, 4>(sb, sms, 4, slab, idx, n_idx, out);
        run<32, 2>(sb, sms, 4, slab, idx, n_idx, out);
    }
    // occupancy / unroll sweep on the L2-resident and the DRAM case
    for (long mb : {64l, 256l}) {
        const long sb = mb << 20;
        run<512, 4>(sb, sms, 8, slab, idx, n_idx / 2, out);
        run<512, 16>(sb, sms, 2, slab, idx, n_idx / 2, out);
        run<128, 16>(sb, sms, 4, slab, idx, n_idx, out);
        run<128, 8>(sb, sms, 8, slab, idx, n_idx, out);
    }
    return 0;
}
