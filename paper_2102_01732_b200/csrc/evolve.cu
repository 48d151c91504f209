// evolve.cu — SET topology evolution on the device (Alg. 2).
//
// Per weight layer that is not dense-capped:
//   1. counts of the sign classes (sign bit 0 / 1, R7) and of occupied alive x alive positions;
//      k_+ = floor(zeta n_+), k_- = floor(zeta n_-) in IEEE double on the host (one multiply, floor)
//   2. selection by radix SELECT (no sort): per sign class s, the k_s-th smallest of the unique
//      63-bit keys  abs_bits(w) << 32 | canonical index  (R5, R6: |w| first, ties by canonical
//      index) is found digit by digit, most significant first -- 8 passes of 8 bits, each a
//      histogram of the entries still matching the class's prefix (integer atomics, exact)
//      followed by a one-block scan that fixes the next digit and the rank left inside it; the
//      prefix state stays on the device (no host round trip between passes).  Then every entry
//      of class s with key <= T_s is removed: exactly k_s of them, the same set the oracle's
//      sort by (|w|, index) takes.
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

// Radix-select state per sign class: the key prefix fixed so far (digits above the current one)
// and the 1-based rank still to find below it.
struct SelState {
    unsigned long long prefix[2];
    unsigned long long rank[2];      // 0: nothing to remove in this class
};
constexpr int SEL_BITS = 8, SEL_BINS = 1 << SEL_BITS, SEL_PASSES = 64 / SEL_BITS;

__device__ __forceinline__ unsigned long long sel_key(uint32_t bits, int64_t k) {
    return ((unsigned long long)(bits & 0x7fffffffu) << 32) | (unsigned long long)k;
}

// pass p: histogram of digit (key >> shift) & 255 over the class's entries whose key agrees with
// its prefix above that digit
__global__ void __launch_bounds__(TPB) select_hist_kernel(const float* __restrict__ val, int64_t nnz, int shift,
                                                          const SelState* __restrict__ st,
                                                          unsigned long long* __restrict__ hist) {
    __shared__ unsigned int sh[2 * SEL_BINS];
    for (int t = threadIdx.x; t < 2 * SEL_BINS; t += blockDim.x) sh[t] = 0;
    __syncthreads();
    const unsigned long long p0 = st->prefix[0], p1 = st->prefix[1];
    const bool a0 = st->rank[0] != 0, a1 = st->rank[1] != 0;
    const int hs = shift + SEL_BITS;          // bits above the digit
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t bits = __float_as_uint(val[k]);
        const int c = bits >> 31;
        const unsigned long long key = sel_key(bits, k);
        const bool on = c ? a1 : a0;
        const unsigned long long hi = hs >= 64 ? 0ull : key >> hs;
        const int bin = (on && hi == (c ? p1 : p0)) ? c * SEL_BINS + (int)((key >> shift) & (SEL_BINS - 1)) : -1;
        // warp-aggregated: most keys of a pass share a few digits (the exponent bits first)
        const unsigned m = __match_any_sync(__activemask(), bin);
        if (bin >= 0 && (__ffs(m) - 1) == (int)(threadIdx.x & 31)) atomicAdd(&sh[bin], (unsigned)__popc(m));
    }
    __syncthreads();
    for (int t = threadIdx.x; t < 2 * SEL_BINS; t += blockDim.x)
        if (sh[t]) atomicAdd(&hist[t], (unsigned long long)sh[t]);
}

// one block: per class, the digit whose cumulative count reaches the rank; extend the prefix,
// keep the rank left inside that digit, clear the histogram for the next pass
__global__ void select_scan_kernel(SelState* st, unsigned long long* hist) {
    const int c = threadIdx.x;
    if (c < 2 && st->rank[c] != 0) {
        unsigned long long r = st->rank[c], below = 0;
        int d = 0;
        for (; d < SEL_BINS; ++d) {
            const unsigned long long n = hist[c * SEL_BINS + d];
            if (below + n >= r) break;
            below += n;
        }
        st->prefix[c] = (st->prefix[c] << SEL_BITS) | (unsigned long long)d;
        st->rank[c] = r - below;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < 2 * SEL_BINS; t += blockDim.x) hist[t] = 0;
}

// after the last pass prefix[c] is the k_c-th smallest key T_c: remove every key <= T_c
__global__ void removal_flags_kernel(const float* __restrict__ val, int64_t nnz, const SelState* __restrict__ st,
                                     const unsigned long long* __restrict__ want, uint8_t* __restrict__ flags) {
    const unsigned long long t0 = st->prefix[0], t1 = st->prefix[1];
    const bool a0 = want[0] != 0, a1 = want[1] != 0;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t bits = __float_as_uint(val[k]);
        const int c = bits >> 31;
        const unsigned long long key = sel_key(bits, k);
        flags[k] = (c ? (a1 && key <= t1) : (a0 && key <= t0)) ? 1 : 0;
    }
}

__global__ void select_init_kernel(SelState* st, unsigned long long* want, unsigned long long* hist,
                                   unsigned long long kp, unsigned long long kn) {
    st->prefix[0] = st->prefix[1] = 0;
    st->rank[0] = kp;
    st->rank[1] = kn;
    want[0] = kp;
    want[1] = kn;
    for (int t = 0; t < 2 * SEL_BINS; ++t) hist[t] = 0;
}

// flags[k] = 1 for the kp smallest positive-class and kn smallest negative-class keys
int radix_select_flags(smlp_handle* h, const float* val, int64_t nnz, int64_t kp, int64_t kn, uint8_t* flags) {
    const size_t ws = sizeof(SelState) + 2 * sizeof(unsigned long long) + 2 * SEL_BINS * sizeof(unsigned long long);
    char* buf = (char*)tmp_alloc(h, ws);
    if (!buf) return set_err(h, SMLP_E_NOMEM, "selection workspace");
    SelState* st = (SelState*)buf;
    unsigned long long* want = (unsigned long long*)(buf + sizeof(SelState));
    unsigned long long* hist = want + 2;
    select_init_kernel<<<1, 1, 0, h->stream>>>(st, want, hist, (unsigned long long)kp, (unsigned long long)kn);
    SMLP_CK_LAUNCH(h, "select_init_kernel");
    const int grid = launch_grid(h, nnz, TPB);
    for (int p = 0; p < SEL_PASSES; ++p) {
        const int shift = 64 - SEL_BITS * (p + 1);
        select_hist_kernel<<<grid, TPB, 0, h->stream>>>(val, nnz, shift, st, hist);
        SMLP_CK_LAUNCH(h, "select_hist_kernel");
        select_scan_kernel<<<1, 64, 0, h->stream>>>(st, hist);
        SMLP_CK_LAUNCH(h, "select_scan_kernel");
    }
    removal_flags_kernel<<<grid, TPB, 0, h->stream>>>(val, nnz, st, want, flags);
    SMLP_CK_LAUNCH(h, "removal_flags_kernel");
    tmp_free(h, buf, ws);
    return SMLP_OK;
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
        // --- selection (radix select of the k_+ / k_- smallest keys per sign class)
        const size_t n = (size_t)nnz;
        uint8_t* flags = (uint8_t*)tmp_alloc(h, n);
        if (!flags) return set_err(h, SMLP_E_NOMEM, "selection flags");
        SMLP_TRY(radix_select_flags(h, Ly.val, nnz, kp, kn, flags));
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
        tmp_free(h, flags, n);
        if (removed) removed[l - 1] = R;
    }
    h->version++;
    h->trace_valid = false;
    return SMLP_OK;
}

}  // namespace smlp
