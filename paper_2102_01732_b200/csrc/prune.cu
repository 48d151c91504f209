// prune.cu — neuron importance (Eq. 4) and Importance Pruning
// (Alg. 2).
//
//   importance_kernel  one thread per neuron j: I_j = sum_i |w_ij| walking the output-major mirror
//                      row j, whose entries are in ascending i (stable sort), as a sequential fp64
//                      sum — the same order and rounding as the oracle, so bit-identical
//   threshold_kernel   type-7 percentile of the sorted alive importances with explicit IEEE
//                      double ops (no FMA contraction: __dadd_rn / __dmul_rn)
//   kill               alive j with I_j < t; incoming column of W^(h) and outgoing row of
//                      W^(h+1) compacted away; all decisions from one snapshot (R19)
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include "smlp_internal.cuh"

namespace smlp {
namespace {

constexpr int TPB = 256;

__global__ void importance_kernel(const int32_t* __restrict__ mrow_ptr, const int32_t* __restrict__ mperm,
                                  const float* __restrict__ val, int64_t n_out, double* __restrict__ I) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n_out; j += (int64_t)gridDim.x * blockDim.x) {
        double acc = 0.0;
        const int32_t e = mrow_ptr[j + 1];
        for (int32_t t = mrow_ptr[j]; t < e; ++t) acc = __dadd_rn(acc, fabs((double)val[mperm[t]]));
        I[j] = acc;
    }
}

__global__ void threshold_kernel(const double* __restrict__ sorted, int64_t n, double rho, double* __restrict__ t_out) {
    const double hh = __ddiv_rn(__dmul_rn((double)(n - 1), rho), 100.0);
    const int64_t lo = (int64_t)floor(hh);
    const int64_t hi = lo + 1 < n - 1 ? lo + 1 : n - 1;
    const double a = sorted[lo], b = sorted[hi];
    *t_out = __dadd_rn(a, __dmul_rn(__dsub_rn(hh, (double)lo), __dsub_rn(b, a)));
}

__global__ void dead_kernel(const double* __restrict__ I, const uint8_t* __restrict__ alive, int64_t n,
                            const double* __restrict__ t, uint8_t* __restrict__ dead, int32_t* __restrict__ count) {
    const double th = *t;
    int32_t c = 0;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const bool d = alive[j] && I[j] < th;
        dead[j] = d ? 1 : 0;
        c += d ? 1 : 0;
    }
    typedef cub::BlockReduce<int32_t, TPB> BR;
    __shared__ typename BR::TempStorage ts;
    const int32_t s = BR(ts).Sum(c);
    if (threadIdx.x == 0) atomicAdd(count, s);
}

__global__ void flags_by_col_kernel(const int32_t* __restrict__ col, int64_t nnz, const uint8_t* __restrict__ dead,
                                    uint8_t* __restrict__ flags) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x)
        flags[k] = dead[col[k]];
}

__global__ void kill_kernel(const uint8_t* __restrict__ dead, int64_t n, uint8_t* __restrict__ alive) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
        if (dead[j]) alive[j] = 0;
}

}  // namespace

int run_importance(smlp_handle* h, int l, double* out_dev) {
    const Layer& Ly = h->layers[l - 2];
    importance_kernel<<<launch_grid(h, Ly.n_out, TPB), TPB, 0, h->stream>>>(Ly.mrow_ptr, Ly.mperm, Ly.val, Ly.n_out,
                                                                             out_dev);
    SMLP_CK_LAUNCH(h, "importance_kernel");
    return SMLP_OK;
}

int run_prune(smlp_handle* h, double rho, int flags, int64_t* pruned, int64_t* removed) {
    const int L = h->L;
    std::vector<double*> I(L + 1, nullptr);
    std::vector<uint8_t*> dead(L + 1, nullptr);
    std::vector<bool> decided(L + 1, false);
    std::vector<int64_t> Dv(L + 1, 0);
    for (int l = 0; l < L; ++l) {
        if (pruned) pruned[l] = 0;
        if (removed) removed[l] = 0;
    }
    // 1. snapshot of all importances
    for (int hl = 2; hl <= L - 1; ++hl) {
        I[hl] = (double*)tmp_alloc(h, sizeof(double) * (size_t)h->sizes[hl - 1]);
        if (!I[hl]) return set_err(h, SMLP_E_NOMEM, "importance buffer");
        SMLP_TRY(run_importance(h, hl, I[hl]));
    }
    // 2. per-layer thresholds and decisions
    for (int hl = 2; hl <= L - 1; ++hl) {
        const int64_t n = h->sizes[hl - 1];
        const int64_t na = h->alive_h[hl];
        if (na == 0) continue;
        double* Ia = (double*)tmp_alloc(h, sizeof(double) * (size_t)n * 2);
        int64_t* nsel = (int64_t*)tmp_alloc(h, 64);
        double* t = (double*)tmp_alloc(h, 64);
        int32_t* cnt = (int32_t*)tmp_alloc(h, 64);
        dead[hl] = (uint8_t*)tmp_alloc(h, (size_t)n);
        if (!Ia || !nsel || !t || !cnt || !dead[hl]) return set_err(h, SMLP_E_NOMEM, "prune workspace");
        double* Is = Ia + n;
        size_t tb1 = 0, tb2 = 0;
        cub::DeviceSelect::Flagged(nullptr, tb1, I[hl], h->alive[hl], Ia, nsel, n, h->stream);
        cub::DeviceRadixSort::SortKeys(nullptr, tb2, Ia, Is, na, 0, 64, h->stream);
        const size_t tb = std::max(tb1, tb2);
        void* tmp = tmp_alloc(h, tb);
        if (!tmp) return set_err(h, SMLP_E_NOMEM, "cub temp");
        SMLP_CK(h, cub::DeviceSelect::Flagged(tmp, tb1, I[hl], h->alive[hl], Ia, nsel, n, h->stream));
        SMLP_CK(h, cub::DeviceRadixSort::SortKeys(tmp, tb2, Ia, Is, na, 0, 64, h->stream));
        threshold_kernel<<<1, 1, 0, h->stream>>>(Is, na, rho, t);
        SMLP_CK_LAUNCH(h, "threshold_kernel");
        SMLP_CK(h, cudaMemsetAsync(cnt, 0, 4, h->stream));
        dead_kernel<<<launch_grid(h, n, TPB), TPB, 0, h->stream>>>(I[hl], h->alive[hl], n, t, dead[hl], cnt);
        SMLP_CK_LAUNCH(h, "dead_kernel");
        int32_t D = 0;
        SMLP_CK(h, cudaMemcpyAsync(&D, cnt, 4, cudaMemcpyDeviceToHost, h->stream));
        SMLP_CK(h, cudaStreamSynchronize(h->stream));
        tmp_free(h, tmp, tb);
        tmp_free(h, Ia, sizeof(double) * (size_t)n * 2);
        tmp_free(h, nsel, 64);
        tmp_free(h, t, 64);
        tmp_free(h, cnt, 64);
        if (D == na) {
            if (pruned) pruned[hl - 1] = -1;        // would kill every alive neuron: skip
            continue;
        }
        decided[hl] = D > 0;
        Dv[hl] = D;
        if (pruned) pruned[hl - 1] = D;
    }
    // 3. apply all decisions
    for (int hl = 2; hl <= L - 1; ++hl) {
        if (!decided[hl]) continue;
        const int64_t n = h->sizes[hl - 1];
        Layer& Lin = h->layers[hl - 2];
        {
            const int64_t before = Lin.nnz;
            uint8_t* fl = (uint8_t*)tmp_alloc(h, (size_t)std::max<int64_t>(before, 1));
            if (!fl) return set_err(h, SMLP_E_NOMEM, "flags");
            if (before > 0) {
                flags_by_col_kernel<<<launch_grid(h, before, TPB), TPB, 0, h->stream>>>(Lin.col, before, dead[hl], fl);
                SMLP_CK_LAUNCH(h, "flags_by_col_kernel");
            }
            SMLP_TRY(compact_layer(h, Lin, fl));
            tmp_free(h, fl, (size_t)std::max<int64_t>(before, 1));
            if (removed) removed[hl - 1] += before - Lin.nnz;
        }
        if (flags & SMLP_PRUNE_OUTGOING) {
            Layer& Lout = h->layers[hl - 1];
            const int64_t before = Lout.nnz;
            uint8_t* fl = (uint8_t*)tmp_alloc(h, (size_t)std::max<int64_t>(before, 1));
            if (!fl) return set_err(h, SMLP_E_NOMEM, "flags");
            if (before > 0) {
                flags_by_col_kernel<<<launch_grid(h, before, TPB), TPB, 0, h->stream>>>(Lout.rowid, before, dead[hl],
                                                                                         fl);
                SMLP_CK_LAUNCH(h, "flags_by_col_kernel");
            }
            SMLP_TRY(compact_layer(h, Lout, fl));
            tmp_free(h, fl, (size_t)std::max<int64_t>(before, 1));
            if (removed) removed[hl] += before - Lout.nnz;
        }
        kill_kernel<<<launch_grid(h, n, TPB), TPB, 0, h->stream>>>(dead[hl], n, h->alive[hl]);
        SMLP_CK_LAUNCH(h, "kill_kernel");
        h->alive_h[hl] -= Dv[hl];
    }
    SMLP_CK(h, cudaStreamSynchronize(h->stream));
    for (int hl = 2; hl <= L - 1; ++hl) {
        if (I[hl]) tmp_free(h, I[hl], sizeof(double) * (size_t)h->sizes[hl - 1]);
        if (dead[hl]) tmp_free(h, dead[hl], (size_t)h->sizes[hl - 1]);
    }
    h->version++;
    h->trace_valid = false;
    return SMLP_OK;
}

}  // namespace smlp
