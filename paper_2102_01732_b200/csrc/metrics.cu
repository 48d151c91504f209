// metrics.cu — gradient flow: the squared L2 norm of the gradient of an
// unfused backward, sum over layers of sum_k g_k^2 over the existing connections (k < nnz of the
// layer) plus sum gb^2 over the biases ("the first-order approximation of the
// decrease in the loss expected after a gradient step").
//
// Deterministic: a fixed grid of GF_BLOCKS blocks, each summing a fixed strided share in fp64
// with a fixed tree, then one block summing the block partials in order.  No atomics.
#include <cuda_runtime.h>

#include "smlp_internal.cuh"

namespace smlp {
namespace {

constexpr int GF_BLOCKS = 592;
constexpr int GF_THREADS = 256;

// ranges: [lo, hi) pairs of the view (one per weight layer: its nnz entries; one for the biases)
struct GfRanges {
    int64_t lo[SMLP_MAX_LAYERS + 1];
    int64_t hi[SMLP_MAX_LAYERS + 1];                 // end of the range when meta is NULL
    const LayerMeta* meta[SMLP_MAX_LAYERS + 1];      // weight layer: the range ends at lo + device nnz
    int count;
};

__global__ void __launch_bounds__(GF_THREADS) gf_partial_kernel(const float* __restrict__ g, GfRanges R,
                                                                double* __restrict__ part) {
    __shared__ double red[GF_THREADS];
    double s = 0.0;
    for (int r = 0; r < R.count; ++r) {
        const int64_t lo = R.lo[r];
        const int64_t hi = R.meta[r] ? lo + R.meta[r]->nnz : R.hi[r];
        for (int64_t k = lo + (int64_t)blockIdx.x * GF_THREADS + threadIdx.x; k < hi; k += (int64_t)GF_BLOCKS * GF_THREADS) {
            const double v = (double)g[k];
            s = fma(v, v, s);
        }
    }
    red[threadIdx.x] = s;
    __syncthreads();
    for (int w = GF_THREADS / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

__global__ void __launch_bounds__(32) gf_final_kernel(const double* __restrict__ part, double* __restrict__ out) {
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int b = 0; b < GF_BLOCKS; ++b) s += part[b];
        *out = s;
    }
}

}  // namespace
}  // namespace smlp

int sparse_mlp_gradient_flow(smlp_handle* h, double* out_host) {
    using namespace smlp;
    if (!h || !out_host) return SMLP_E_ARG;
    if (!h->grads_pending) return set_err(h, SMLP_E_STATE, "gradient_flow needs the gradient of an unfused backward");
    GfRanges R{};
    R.count = 0;
    for (auto& Ly : h->layers) {
        R.lo[R.count] = Ly.val_off;
        R.meta[R.count] = Ly.meta;
        R.hi[R.count] = 0;
        ++R.count;
    }
    R.lo[R.count] = h->bias_base;
    R.meta[R.count] = nullptr;
    R.hi[R.count] = h->param_count;
    ++R.count;
    double* buf = (double*)tmp_alloc(h, sizeof(double) * (GF_BLOCKS + 1));
    if (!buf) return set_err(h, SMLP_E_NOMEM, "gradient_flow scratch");
    gf_partial_kernel<<<GF_BLOCKS, GF_THREADS, 0, h->stream>>>(h->grad, R, buf);
    SMLP_CK_LAUNCH(h, "gf_partial_kernel");
    gf_final_kernel<<<1, 32, 0, h->stream>>>(buf, buf + GF_BLOCKS);
    SMLP_CK_LAUNCH(h, "gf_final_kernel");
    SMLP_CK(h, cudaMemcpyAsync(out_host, buf + GF_BLOCKS, sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    SMLP_CK(h, cudaStreamSynchronize(h->stream));
    tmp_free(h, buf, sizeof(double) * (GF_BLOCKS + 1));
    return SMLP_OK;
}
