// evolve.cu — SET topology evolution on the device (Alg. 2).
//
// Per weight layer that is not dense-capped:
//   1. counts of the sign classes (sign bit 0 / 1, R7) and of occupied alive x alive positions;
//      k_+ = floor(zeta n_+), k_- = floor(zeta n_-) in IEEE double on the host (one multiply, floor)
//   2. selection: one radix sort of 64-bit keys  sign << 63 | abs_bits(w) << 32 | canonical index;
//      positives come first ordered by |w| then index, then negatives likewise, so the removed
//      entries are sorted[0, k_+) and sorted[n_+, n_+ + k_-)  (R5, R6: ties by canonical index)
//   3. regrowth: the first R = k_+ + k_- distinct REGROW-stream candidates outside the pre-call
//      support between alive neurons (R8), values from the init scheme (R4)
//   4. merge survivors and additions into the canonical CSR, rebuild mirror + work lists
// A layer with fewer free positions than R is left unchanged (R9).  Everything is integer
// arithmetic on IEEE bit patterns, so the result is bit-identical to the oracle's.
#include <cuda_runtime.h>

#include <cmath>
#include <cub/cub.cuh>

#include "smlp_internal.cuh"

namespace smlp {
namespace {

constexpr int TPB = 256;

__global__ void evolve_counts_kernel(const float* __restrict__ val, const int32_t* __restrict__ rowid,
                                     const int32_t* __restrict__ col, const uint8_t* __restrict__ alive_in,
                                     const uint8_t* __restrict__ alive_out, int64_t nnz,
                                     unsigned long long* __restrict__ out2) {
    unsigned long long pos = 0, occ = 0;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t bits = __float_as_uint(val[k]);
        pos += (bits >> 31) == 0 ? 1ull : 0ull;
        occ += (alive_in[rowid[k]] && alive_out[col[k]]) ? 1ull : 0ull;
    }
    typedef cub::BlockReduce<unsigned long long, TPB> BR;
    __shared__ typename BR::TempStorage t1, t2;
    const unsigned long long sp = BR(t1).Sum(pos);
    const unsigned long long so = BR(t2).Sum(occ);
    if (threadIdx.x == 0) {
        atomicAdd(out2, sp);        // integer atomics: exact and order-independent
        atomicAdd(out2 + 1, so);
    }
}

__global__ void selection_keys_kernel(const float* __restrict__ val, int64_t nnz, uint64_t* __restrict__ keys) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t bits = __float_as_uint(val[k]);
        keys[k] = ((uint64_t)(bits >> 31) << 63) | ((uint64_t)(bits & 0x7fffffffu) << 32) | (uint64_t)k;
    }
}

__global__ void removal_flags_kernel(const uint64_t* __restrict__ sorted, int64_t npos, int64_t kp, int64_t kn,
                                     uint8_t* __restrict__ flags) {
    const int64_t R = kp + kn;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < R; r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = r < kp ? r : npos + (r - kp);
        flags[sorted[t] & 0xffffffffull] = 1;
    }
}

}  // namespace

int run_evolve(smlp_handle* h, double zeta, uint64_t e, int64_t* removed) {
    for (int l = 2; l <= h->L; ++l) {
        Layer& Ly = h->layers[l - 2];
        if (removed) removed[l - 1] = -1;
        if (Ly.dense) continue;
        const int64_t nnz = Ly.nnz;
        unsigned long long* cnt = (unsigned long long*)tmp_alloc(h, 16);
        if (!cnt) return set_err(h, SMLP_E_NOMEM, "evolve counts");
        SMLP_CK(h, cudaMemsetAsync(cnt, 0, 16, h->stream));
        if (nnz > 0) {
            evolve_counts_kernel<<<launch_grid(h, nnz, TPB), TPB, 0, h->stream>>>(
                Ly.val, Ly.rowid, Ly.col, h->alive[l - 1], h->alive[l], nnz, cnt);
            SMLP_CK_LAUNCH(h, "evolve_counts_kernel");
        }
        unsigned long long c2[2];
        SMLP_CK(h, cudaMemcpyAsync(c2, cnt, 16, cudaMemcpyDeviceToHost, h->stream));
        SMLP_CK(h, cudaStreamSynchronize(h->stream));
        tmp_free(h, cnt, 16);
        const int64_t npos = (int64_t)c2[0], nneg = nnz - npos, occ = (int64_t)c2[1];
        const int64_t kp = (int64_t)std::floor(zeta * (double)npos);
        const int64_t kn = (int64_t)std::floor(zeta * (double)nneg);
        const int64_t R = kp + kn;
        const int64_t A = h->alive_h[l - 1] * h->alive_h[l] - occ;
        if (R == 0) {
            if (removed) removed[l - 1] = 0;
            continue;
        }
        if (A < R) continue;                       // skip rule: saturated layer stays unchanged
        // --- selection
        const size_t n = (size_t)nnz;
        uint64_t* keys = (uint64_t*)tmp_alloc(h, 2 * n * sizeof(uint64_t));
        uint8_t* flags = (uint8_t*)tmp_alloc(h, n);
        if (!keys || !flags) return set_err(h, SMLP_E_NOMEM, "selection workspace");
        uint64_t* sorted = keys + n;
        selection_keys_kernel<<<launch_grid(h, nnz, TPB), TPB, 0, h->stream>>>(Ly.val, nnz, keys);
        SMLP_CK_LAUNCH(h, "selection_keys_kernel");
        size_t tb = 0;
        cub::DeviceRadixSort::SortKeys(nullptr, tb, keys, sorted, (int64_t)nnz, 0, 64, h->stream);
        void* tmp = tmp_alloc(h, tb);
        if (!tmp) return set_err(h, SMLP_E_NOMEM, "radix temp");
        SMLP_CK(h, cub::DeviceRadixSort::SortKeys(tmp, tb, keys, sorted, (int64_t)nnz, 0, 64, h->stream));
        SMLP_CK(h, cudaMemsetAsync(flags, 0, n, h->stream));
        removal_flags_kernel<<<launch_grid(h, R, TPB), TPB, 0, h->stream>>>(sorted, npos, kp, kn, flags);
        SMLP_CK_LAUNCH(h, "removal_flags_kernel");
        // --- regrowth (pre-call support still in place)
        uint64_t* add_pos = (uint64_t*)tmp_alloc(h, (size_t)R * sizeof(uint64_t));
        float* add_val = (float*)tmp_alloc(h, (size_t)R * sizeof(float));
        if (!add_pos || !add_val) return set_err(h, SMLP_E_NOMEM, "regrowth buffers");
        SMLP_TRY(first_distinct_candidates(h, Ly, P_REGROW, (uint32_t)e, R, true, h->alive[l - 1], h->alive[l], A,
                                           add_pos, add_val));
        // --- merge + rebuild
        SMLP_TRY(merge_layer(h, Ly, flags, add_pos, add_val, R));
        tmp_free(h, add_pos, (size_t)R * sizeof(uint64_t));
        tmp_free(h, add_val, (size_t)R * sizeof(float));
        tmp_free(h, tmp, tb);
        tmp_free(h, keys, 2 * n * sizeof(uint64_t));
        tmp_free(h, flags, n);
        if (removed) removed[l - 1] = R;
    }
    h->version++;
    h->trace_valid = false;
    return SMLP_OK;
}

}  // namespace smlp
