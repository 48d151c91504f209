// union.cu — WASAP phase-2 model averaging over the UNION of K supports (
// Alg. 1, Eq. 2; SPEC S:282-290 average_models).
//
// After phase 2 the K replicas have evolved their topologies independently.  For one weight layer
// the caller gathers every replica's (position, value) list (sorted canonical positions
// i * n_out + j, rank order) into one device array; then, identically on every replica:
//   1. stable radix sort of the positions (equal positions keep rank order);
//   2. union: one entry per distinct position; its value is the fp32 sum of the present values in
//      rank order (absent = 0, so absent values are simply not added), divided by K in fp32
//      (DESIGN reading R31: both the oracle and this kernel take the value -- and so the selection
//      below -- in exactly this arithmetic);
//   3. re-sparsification to `target` connections (the phase-1 per-layer count): the union entries
//      closest to zero are removed -- 64-bit keys (|w| bits << 32 | union index) sorted ascending,
//      the first U - target removed ("unimportant connections ... are pruned");
//   4. the kept entries (still in position order) become the layer's canonical CSR, momentum 0,
//      and the mirror / work lists are rebuilt.  version += 1.
// Integer decisions only depend on IEEE bit patterns, so every replica ends bit-identical.
#include <cuda_runtime.h>

#include <cub/cub.cuh>
#include <vector>

#include "smlp_internal.cuh"

namespace smlp {
namespace {

constexpr int TPB = 256;

int bits_u64(uint64_t v) {
    int b = 1;
    while (b < 64 && (v >> b) != 0) ++b;
    return b;
}

// Eq. 2 after a SUM allreduce of the param view: theta <- theta_sum / K (fp32, one rounding)
__global__ void divide_kernel(float* __restrict__ p, int64_t n, float K) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        p[k] = __fdiv_rn(p[k], K);
}

// canonical positions i * n_out + j of a layer's entries
__global__ void positions_kernel(const int32_t* __restrict__ rowid, const int32_t* __restrict__ col, int64_t nnz,
                                 int64_t n_out, uint64_t* __restrict__ pos) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x)
        pos[k] = (uint64_t)rowid[k] * (uint64_t)n_out + (uint64_t)col[k];
}

// scratch buffers freed together
struct Scratch {
    smlp_handle* h;
    std::vector<std::pair<void*, size_t>> v;
    void* get(size_t bytes) {
        void* p = tmp_alloc(h, bytes);
        if (p) v.push_back({p, bytes});
        return p;
    }
    ~Scratch() {
        for (auto& e : v) tmp_free(h, e.first, e.second);
    }
};

__global__ void iota64_kernel(int64_t* __restrict__ a, int64_t n) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        a[k] = k;
}

// flags[t] = 1 where a new position starts in the sorted sequence
__global__ void seg_start_kernel(const uint64_t* __restrict__ pos, int64_t n, uint8_t* __restrict__ flags) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
        flags[t] = (t == 0 || pos[t] != pos[t - 1]) ? 1 : 0;
}

// one thread per union entry: fp32 sum of its (<= K) values in rank order, / K; selection key
__global__ void union_values_kernel(const uint64_t* __restrict__ pos_sorted, const int64_t* __restrict__ src,
                                    const float* __restrict__ val_all, const int64_t* __restrict__ starts,
                                    const int64_t* __restrict__ nunion, int64_t total, int K,
                                    uint64_t* __restrict__ upos, float* __restrict__ uval,
                                    uint64_t* __restrict__ keys) {
    const int64_t U = *nunion;
    for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < U; u += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t0 = starts[u], t1 = u + 1 < U ? starts[u + 1] : total;
        float s = val_all[src[t0]];
        for (int64_t t = t0 + 1; t < t1; ++t) s = __fadd_rn(s, val_all[src[t]]);
        const float avg = __fdiv_rn(s, (float)K);
        upos[u] = pos_sorted[t0];
        uval[u] = avg;
        keys[u] = ((uint64_t)(__float_as_uint(avg) & 0x7fffffffu) << 32) | (uint64_t)u;
    }
}

__global__ void removal_from_keys_kernel(const uint64_t* __restrict__ sorted_keys, int64_t nremove,
                                         uint8_t* __restrict__ keep) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nremove; r += (int64_t)gridDim.x * blockDim.x)
        keep[sorted_keys[r] & 0xffffffffull] = 0;
}

}  // namespace
}  // namespace smlp

int sparse_mlp_union_average_layer(smlp_handle* h, int32_t l, int32_t K, const uint64_t* pos_all,
                                   const float* val_all, int64_t total, int64_t target, int64_t* kept) {
    using namespace smlp;
    if (!h || l < 2 || l > h->L || K < 1 || total < 0 || target < 0 || (total > 0 && (!pos_all || !val_all)))
        return SMLP_E_ARG;
    Layer& Ly = h->layers[l - 2];
    if (target > Ly.cap) return set_err(h, SMLP_E_ARG, "union average: target exceeds the layer capacity");
    const int64_t T = total;
    const int endbit = bits_u64((uint64_t)Ly.n_in * (uint64_t)Ly.n_out);
    Scratch S{h, {}};
    const size_t Tn = (size_t)std::max<int64_t>(T, 1);
    uint64_t* pos_s = (uint64_t*)S.get(sizeof(uint64_t) * Tn);
    int64_t* idx = (int64_t*)S.get(sizeof(int64_t) * Tn);
    int64_t* src = (int64_t*)S.get(sizeof(int64_t) * Tn);
    uint8_t* flags = (uint8_t*)S.get(Tn);
    int64_t* starts = (int64_t*)S.get(sizeof(int64_t) * Tn);
    int64_t* nsel = (int64_t*)S.get(sizeof(int64_t) * 2);
    if (!pos_s || !idx || !src || !flags || !starts || !nsel) return set_err(h, SMLP_E_NOMEM, "union average workspace");
    int64_t U = 0;
    if (T > 0) {
        iota64_kernel<<<launch_grid(h, T, TPB), TPB, 0, h->stream>>>(idx, T);
        SMLP_CK_LAUNCH(h, "iota64_kernel");
        size_t tb = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tb, pos_all, pos_s, idx, src, T, 0, endbit, h->stream);
        void* tmp = S.get(tb);
        if (!tmp) return set_err(h, SMLP_E_NOMEM, "radix temp");
        SMLP_CK(h, cub::DeviceRadixSort::SortPairs(tmp, tb, pos_all, pos_s, idx, src, T, 0, endbit, h->stream));
        seg_start_kernel<<<launch_grid(h, T, TPB), TPB, 0, h->stream>>>(pos_s, T, flags);
        SMLP_CK_LAUNCH(h, "seg_start_kernel");
        size_t tb2 = 0;
        cub::DeviceSelect::Flagged(nullptr, tb2, idx, flags, starts, nsel, T, h->stream);
        void* tmp2 = S.get(tb2);
        if (!tmp2) return set_err(h, SMLP_E_NOMEM, "select temp");
        // idx is 0..T-1 again (SortPairs does not modify its inputs), so the selected values are
        // the sorted-sequence indices where a new position starts
        SMLP_CK(h, cub::DeviceSelect::Flagged(tmp2, tb2, idx, flags, starts, nsel, T, h->stream));
        SMLP_CK(h, cudaMemcpyAsync(&U, nsel, sizeof(int64_t), cudaMemcpyDeviceToHost, h->stream));
        SMLP_CK(h, cudaStreamSynchronize(h->stream));
    }
    const int64_t keep_n = std::min<int64_t>(U, target);
    const size_t Un = (size_t)std::max<int64_t>(U, 1);
    uint64_t* upos = (uint64_t*)S.get(sizeof(uint64_t) * Un);
    float* uval = (float*)S.get(sizeof(float) * Un);
    uint64_t* keys = (uint64_t*)S.get(sizeof(uint64_t) * 2 * Un);
    uint8_t* keep = (uint8_t*)S.get(Un);
    uint64_t* kpos = (uint64_t*)S.get(sizeof(uint64_t) * Un);
    float* kval = (float*)S.get(sizeof(float) * Un);
    if (!upos || !uval || !keys || !keep || !kpos || !kval) return set_err(h, SMLP_E_NOMEM, "union buffers");
    if (U > 0) {
        union_values_kernel<<<launch_grid(h, U, TPB), TPB, 0, h->stream>>>(pos_s, src, val_all, starts, nsel, T, K,
                                                                            upos, uval, keys);
        SMLP_CK_LAUNCH(h, "union_values_kernel");
        SMLP_CK(h, cudaMemsetAsync(keep, 1, (size_t)U, h->stream));
        if (U > keep_n) {
            size_t tb = 0;
            uint64_t* ksorted = keys + U;
            cub::DeviceRadixSort::SortKeys(nullptr, tb, keys, ksorted, U, 0, 64, h->stream);
            void* tmp = S.get(tb);
            if (!tmp) return set_err(h, SMLP_E_NOMEM, "radix temp");
            SMLP_CK(h, cub::DeviceRadixSort::SortKeys(tmp, tb, keys, ksorted, U, 0, 64, h->stream));
            removal_from_keys_kernel<<<launch_grid(h, U - keep_n, TPB), TPB, 0, h->stream>>>(ksorted, U - keep_n, keep);
            SMLP_CK_LAUNCH(h, "removal_from_keys_kernel");
        }
        size_t tb = 0;
        cub::DeviceSelect::Flagged(nullptr, tb, upos, keep, kpos, nsel + 1, U, h->stream);
        void* tmp = S.get(tb);
        if (!tmp) return set_err(h, SMLP_E_NOMEM, "select temp");
        SMLP_CK(h, cub::DeviceSelect::Flagged(tmp, tb, upos, keep, kpos, nsel + 1, U, h->stream));
        SMLP_CK(h, cub::DeviceSelect::Flagged(tmp, tb, uval, keep, kval, nsel + 1, U, h->stream));
    }
    SMLP_TRY(csr_from_sorted_positions(h, Ly, kpos, kval, keep_n));
    if (kept) *kept = keep_n;
    h->version++;
    h->trace_valid = false;
    h->grads_pending = false;
    return SMLP_OK;
}

int sparse_mlp_export_positions(smlp_handle* h, int32_t l, uint64_t* pos_dev, float* val_dev) {
    using namespace smlp;
    if (!h || l < 2 || l > h->L) return SMLP_E_ARG;
    Layer& Ly = h->layers[l - 2];
    if (Ly.nnz == 0) return SMLP_OK;
    if (!pos_dev || !val_dev) return SMLP_E_ARG;
    positions_kernel<<<launch_grid(h, Ly.nnz, TPB), TPB, 0, h->stream>>>(Ly.rowid, Ly.col, Ly.nnz, Ly.n_out, pos_dev);
    SMLP_CK_LAUNCH(h, "positions_kernel");
    SMLP_CK(h, cudaMemcpyAsync(val_dev, Ly.val, sizeof(float) * (size_t)Ly.nnz, cudaMemcpyDeviceToDevice, h->stream));
    return SMLP_OK;
}

namespace smlp {
namespace {

// g_now[k] = stale gradient at the position of current entry k, 0 if that position was not in the
// stale support (binary search in the sorted stale positions)
__global__ void retain_kernel(const int32_t* __restrict__ rowid, const int32_t* __restrict__ col, int64_t nnz,
                              int64_t n_out, const uint64_t* __restrict__ spos, const float* __restrict__ sg,
                              int64_t ns, float* __restrict__ g_now, unsigned long long* __restrict__ hits) {
    unsigned long long h = 0;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t p = (uint64_t)rowid[k] * (uint64_t)n_out + (uint64_t)col[k];
        int64_t lo = 0, hi = ns;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (spos[mid] < p) lo = mid + 1;
            else hi = mid;
        }
        const bool found = lo < ns && spos[lo] == p;
        g_now[k] = found ? sg[lo] : 0.f;
        h += found ? 1ull : 0ull;
    }
    if (h) atomicAdd(hits, h);   // integer: exact and order-independent
}

}  // namespace
}  // namespace smlp

int sparse_mlp_retain_valid_updates(smlp_handle* h, int32_t l, const uint64_t* stale_pos, const float* stale_g,
                                    int64_t n_stale, int64_t* retained) {
    using namespace smlp;
    if (!h || l < 2 || l > h->L || n_stale < 0 || (n_stale > 0 && (!stale_pos || !stale_g))) return SMLP_E_ARG;
    Layer& Ly = h->layers[l - 2];
    unsigned long long* cnt = (unsigned long long*)tmp_alloc(h, sizeof(unsigned long long));
    if (!cnt) return set_err(h, SMLP_E_NOMEM, "retain counter");
    SMLP_CK(h, cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), h->stream));
    if (Ly.nnz > 0) {
        retain_kernel<<<launch_grid(h, Ly.nnz, TPB), TPB, 0, h->stream>>>(Ly.rowid, Ly.col, Ly.nnz, Ly.n_out, stale_pos,
                                                                          stale_g, n_stale, Ly.grad, cnt);
        SMLP_CK_LAUNCH(h, "retain_kernel");
    }
    unsigned long long c = 0;
    SMLP_CK(h, cudaMemcpyAsync(&c, cnt, sizeof(c), cudaMemcpyDeviceToHost, h->stream));
    SMLP_CK(h, cudaStreamSynchronize(h->stream));
    tmp_free(h, cnt, sizeof(unsigned long long));
    if (retained) *retained = (int64_t)c;
    h->grads_pending = true;    // the caller applies it with sparse_mlp_step (biases: its grad view slice)
    return SMLP_OK;
}

int sparse_mlp_params_averaged(smlp_handle* h, int32_t K, int32_t biases_only) {
    using namespace smlp;
    if (!h) return SMLP_E_ARG;
    if (K < 1) return set_err(h, SMLP_E_ARG, "K must be >= 1");
    const int64_t lo = biases_only ? h->bias_base : 0;
    const int64_t n = h->param_count - lo;
    if (K > 1 && n > 0) {
        divide_kernel<<<launch_grid(h, n, TPB), TPB, 0, h->stream>>>(h->param + lo, n, (float)K);
        SMLP_CK_LAUNCH(h, "divide_kernel");
    }
    if (!biases_only)
        for (auto& Ly : h->layers) SMLP_TRY(refresh_mirror_values(h, Ly));
    return SMLP_OK;
}
