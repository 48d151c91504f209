// topology.cu — building and editing the sparse topology on the device.
//
//   first_distinct_candidates   "the first R distinct valid candidates of a Philox stream" (R2, R8):
//                               generate C candidates, stable radix sort by position, keep the first
//                               occurrence of each position, rank survivors in stream order, take R.
//                               Used by ER initialisation (G(n, M)) and SET regrowth
//                               (Alg. 2).
//   merge_layer                 new canonical CSR = survivors (flag 0) U sorted additions, by a
//                               merge-path of binary searches (no sort); survivors keep (w, v).
//   rebuild_derived             rowid, output-major mirror (stable radix sort by column keeps i
//                               ascending inside a column), and the forward/backward segment lists.
//
// Everything is integer work with deterministic results; only small counts are read back.
#include <cuda_runtime.h>

#include <algorithm>
#include <cub/cub.cuh>

#include "smlp_internal.cuh"

namespace smlp {

int launch_grid(const smlp_handle* h, int64_t items, int threads) {
    const int64_t need = (items + threads - 1) / threads;
    return (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)h->num_sms * 32));
}

namespace {

constexpr int TPB = 256;

template <typename T>
__device__ __forceinline__ int64_t lower_bound_dev(const T* a, int64_t n, T key) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (a[mid] < key) lo = mid + 1; else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ bool in_row(const int32_t* col, int32_t beg, int32_t end, int32_t j) {
    int32_t lo = beg, hi = end;
    while (lo < hi) {
        const int32_t mid = (lo + hi) >> 1;
        const int32_t c = col[mid];
        if (c < j) lo = mid + 1; else hi = mid;
    }
    return lo < end && col[lo] == j;
}

__global__ void gen_candidates_kernel(uint64_t seed, uint32_t purpose, uint32_t layer, uint32_t c3, int64_t C,
                                      int64_t n_in, int64_t n_out, uint64_t sentinel, bool exclude,
                                      const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                                      const uint8_t* __restrict__ alive_in, const uint8_t* __restrict__ alive_out,
                                      uint64_t* __restrict__ keys, uint32_t* __restrict__ ms) {
    for (int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; m < C; m += (int64_t)gridDim.x * blockDim.x) {
        const uint4 r = rng_stream(seed, purpose, 0, layer, c3, (uint64_t)m);
        const uint32_t i = scale_u32(r.x, (uint64_t)n_in);
        const uint32_t j = scale_u32(r.y, (uint64_t)n_out);
        bool valid = true;
        if (alive_in && !alive_in[i]) valid = false;
        if (alive_out && !alive_out[j]) valid = false;
        if (valid && exclude && in_row(col, row_ptr[i], row_ptr[i + 1], (int32_t)j)) valid = false;
        keys[m] = valid ? (uint64_t)i * (uint64_t)n_out + j : sentinel;
        ms[m] = (uint32_t)m;
    }
}

// first occurrence of each valid position (sorted array; stable sort keeps stream order)
__global__ void flag_first_kernel(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ ms, int64_t C,
                                  uint64_t sentinel, int32_t* __restrict__ first_by_m, uint8_t* __restrict__ first_sorted) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < C; t += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = keys[t];
        const bool f = k != sentinel && (t == 0 || keys[t - 1] != k);
        first_sorted[t] = f ? 1 : 0;
        first_by_m[ms[t]] = f ? 1 : 0;
    }
}

// keep sorted entries that are first occurrences with stream rank < R
__global__ void select_flags_kernel(const uint32_t* __restrict__ ms, const uint8_t* __restrict__ first_sorted,
                                    const int32_t* __restrict__ rank_by_m, int64_t C, int64_t R,
                                    uint8_t* __restrict__ sel) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < C; t += (int64_t)gridDim.x * blockDim.x) {
        sel[t] = (first_sorted[t] && rank_by_m[ms[t]] < R) ? 1 : 0;
    }
}

__global__ void candidate_values_kernel(uint64_t seed, uint32_t purpose, uint32_t layer, uint32_t c3,
                                        const uint32_t* __restrict__ ms, int64_t R, InitParams ip,
                                        float* __restrict__ out) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < R; r += (int64_t)gridDim.x * blockDim.x) {
        const uint4 x = rng_stream(seed, purpose, 0, layer, c3, (uint64_t)ms[r]);
        out[r] = init_value(ip, x.z, x.w);
    }
}

__global__ void dense_fill_kernel(uint64_t seed, uint32_t layer, int64_t n_in, int64_t n_out, InitParams ip,
                                  int32_t* __restrict__ row_ptr, int32_t* __restrict__ col, float* __restrict__ val,
                                  float* __restrict__ mom) {
    const int64_t total = n_in * n_out;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
        const uint4 x = rng_stream(seed, P_INIT_DENSE, 0, layer, 0, (uint64_t)k);
        col[k] = (int32_t)(k % n_out);
        val[k] = init_value(ip, x.z, x.w);
        mom[k] = 0.f;
        if (k % n_out == 0) row_ptr[k / n_out] = (int32_t)k;
        if (k == total - 1) row_ptr[n_in] = (int32_t)total;
    }
}

__global__ void csr_from_pos_kernel(const uint64_t* __restrict__ pos, const float* __restrict__ v, int64_t n,
                                    int64_t n_in, int64_t n_out, int32_t* __restrict__ col, float* __restrict__ val,
                                    float* __restrict__ mom) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        col[k] = (int32_t)(pos[k] % (uint64_t)n_out);
        val[k] = v[k];
        mom[k] = 0.f;
    }
}

__global__ void row_ptr_from_pos_kernel(const uint64_t* __restrict__ pos, int64_t n, int64_t n_in, int64_t n_out,
                                        int32_t* __restrict__ row_ptr) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= n_in; i += (int64_t)gridDim.x * blockDim.x) {
        row_ptr[i] = (int32_t)lower_bound_dev<uint64_t>(pos, n, (uint64_t)i * (uint64_t)n_out);
    }
}

__global__ void rowid_kernel(const int32_t* __restrict__ row_ptr, int64_t n_rows, int64_t nnz, int32_t* __restrict__ rowid) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
        // largest i with row_ptr[i] <= k
        int64_t lo = 0, hi = n_rows;
        while (lo < hi) {
            const int64_t mid = (lo + hi + 1) >> 1;
            if (row_ptr[mid] <= k) lo = mid; else hi = mid - 1;
        }
        rowid[k] = (int32_t)lo;
    }
}

__global__ void iota_kernel(int32_t* __restrict__ a, int64_t n) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        a[k] = (int32_t)k;
}

__global__ void mirror_fill_kernel(const int32_t* __restrict__ perm, const int32_t* __restrict__ rowid,
                                   const float* __restrict__ val, int64_t nnz, int32_t* __restrict__ msrc,
                                   int32_t* __restrict__ minv, float* __restrict__ mval) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nnz; t += (int64_t)gridDim.x * blockDim.x) {
        const int32_t k = perm[t];
        msrc[t] = rowid[k];
        minv[k] = (int32_t)t;
        mval[t] = val[k];
    }
}

__global__ void mrow_ptr_kernel(const int32_t* __restrict__ sorted_col, int64_t nnz, int64_t n_out,
                                int32_t* __restrict__ mrow_ptr) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j <= n_out; j += (int64_t)gridDim.x * blockDim.x)
        mrow_ptr[j] = (int32_t)lower_bound_dev<int32_t>(sorted_col, nnz, (int32_t)j);
}

// segment counts per row: max(1, ceil(len / S)); multi rows use one partial slot per segment
__global__ void seg_count_kernel(const int32_t* __restrict__ ptr, int64_t rows, int32_t* __restrict__ nseg,
                                 int32_t* __restrict__ nmulti, int32_t* __restrict__ nslot) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
        const int32_t len = ptr[r + 1] - ptr[r];
        const int32_t n = len <= SEG_NNZ ? 1 : (len + SEG_NNZ - 1) / SEG_NNZ;
        nseg[r] = n;
        nmulti[r] = n > 1 ? 1 : 0;
        nslot[r] = n > 1 ? n : 0;
    }
}

__global__ void seg_fill_kernel(const int32_t* __restrict__ ptr, int64_t rows, const int32_t* __restrict__ nseg,
                                const int32_t* __restrict__ segoff, const int32_t* __restrict__ moff,
                                const int32_t* __restrict__ slotoff, int4* __restrict__ seg, int4* __restrict__ multi) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
        const int32_t beg = ptr[r], end = ptr[r + 1];
        const int32_t n = nseg[r];
        const int32_t so = segoff[r];
        for (int32_t s = 0; s < n; ++s) {
            const int32_t b = beg + s * SEG_NNZ;
            const int32_t e = min(end, b + SEG_NNZ);
            seg[so + s] = make_int4((int32_t)r, b, e, n > 1 ? slotoff[r] + s : -1);
        }
        if (n > 1) multi[moff[r]] = make_int4((int32_t)r, slotoff[r], n, 0);
    }
}

__global__ void totals_kernel(const int32_t* __restrict__ nseg, const int32_t* __restrict__ segoff,
                              const int32_t* __restrict__ nmulti, const int32_t* __restrict__ moff,
                              const int32_t* __restrict__ nslot, const int32_t* __restrict__ slotoff, int64_t rows,
                              int32_t* __restrict__ out3) {
    out3[0] = segoff[rows - 1] + nseg[rows - 1];
    out3[1] = moff[rows - 1] + nmulti[rows - 1];
    out3[2] = slotoff[rows - 1] + nslot[rows - 1];
}

__global__ void set_meta_kernel(LayerMeta* meta, int32_t nnz, const int32_t* __restrict__ f3, const int32_t* __restrict__ b3) {
    meta->nnz = nnz;
    meta->n_fseg = f3[0];
    meta->n_fmulti = f3[1];
    meta->n_bseg = b3[0];
    meta->n_bmulti = b3[1];
}

// merge-path placement of survivors and additions into the new canonical order
__global__ void merge_survivors_kernel(const int32_t* __restrict__ rowid, const int32_t* __restrict__ col,
                                       const float* __restrict__ val, const float* __restrict__ mom,
                                       const uint8_t* __restrict__ flags, const int32_t* __restrict__ sp,
                                       const uint64_t* __restrict__ add_pos, int64_t R, int64_t nnz, int64_t n_out,
                                       int32_t* __restrict__ ncol, float* __restrict__ nval, float* __restrict__ nmom) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
        if (flags && flags[k]) continue;
        const uint64_t key = (uint64_t)rowid[k] * (uint64_t)n_out + (uint64_t)col[k];
        const int64_t dst = (int64_t)sp[k] + (R ? lower_bound_dev<uint64_t>(add_pos, R, key) : 0);
        ncol[dst] = col[k];
        nval[dst] = val[k];
        nmom[dst] = mom[k];
    }
}

__global__ void merge_additions_kernel(const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                                       const int32_t* __restrict__ sp, const uint64_t* __restrict__ add_pos,
                                       const float* __restrict__ add_val, int64_t R, int64_t n_out,
                                       int32_t* __restrict__ ncol, float* __restrict__ nval, float* __restrict__ nmom) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < R; r += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t p = add_pos[r];
        const int64_t i = (int64_t)(p / (uint64_t)n_out);
        const int32_t j = (int32_t)(p % (uint64_t)n_out);
        const int32_t beg = row_ptr[i], end = row_ptr[i + 1];
        int32_t lo = beg, hi = end;
        while (lo < hi) {
            const int32_t mid = (lo + hi) >> 1;
            if (col[mid] < j) lo = mid + 1; else hi = mid;
        }
        const int64_t dst = (int64_t)sp[lo] + r;
        ncol[dst] = j;
        nval[dst] = add_val[r];
        nmom[dst] = 0.f;
    }
}

__global__ void merge_row_ptr_kernel(const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ sp,
                                     const uint64_t* __restrict__ add_pos, int64_t R, int64_t n_in, int64_t n_out,
                                     int32_t* __restrict__ nrow_ptr) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= n_in; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t adds = R ? lower_bound_dev<uint64_t>(add_pos, R, (uint64_t)i * (uint64_t)n_out) : 0;
        nrow_ptr[i] = (int32_t)((int64_t)sp[row_ptr[i]] + adds);
    }
}

__global__ void survivor_flags_kernel(const uint8_t* __restrict__ flags, int64_t nnz, int32_t* __restrict__ s) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k <= nnz; k += (int64_t)gridDim.x * blockDim.x)
        s[k] = (k < nnz && !(flags && flags[k])) ? 1 : 0;
}

int bits_for(uint64_t v) {
    int b = 1;
    while (b < 64 && (v >> b) != 0) ++b;
    return b;
}

// Build a segment list over rows with pointer array ptr (device, rows+1 entries).
int build_segments(smlp_handle* h, const int32_t* ptr, int64_t rows, int4* seg, int64_t seg_cap, int4* multi,
                   int64_t slot_cap, int32_t* totals3) {
    int32_t* buf = (int32_t*)tmp_alloc(h, sizeof(int32_t) * 6 * (size_t)rows);
    if (!buf) return set_err(h, SMLP_E_NOMEM, "segment workspace");
    int32_t *nseg = buf, *nmulti = buf + rows, *nslot = buf + 2 * rows;
    int32_t *segoff = buf + 3 * rows, *moff = buf + 4 * rows, *slotoff = buf + 5 * rows;
    const int grid = launch_grid(h, rows, TPB);
    seg_count_kernel<<<grid, TPB, 0, h->stream>>>(ptr, rows, nseg, nmulti, nslot);
    SMLP_CK_LAUNCH(h, "seg_count_kernel");
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, nseg, segoff, (int)rows, h->stream);
    void* tmp = tmp_alloc(h, tb);
    if (!tmp) return set_err(h, SMLP_E_NOMEM, "scan temp");
    SMLP_CK(h, cub::DeviceScan::ExclusiveSum(tmp, tb, nseg, segoff, (int)rows, h->stream));
    SMLP_CK(h, cub::DeviceScan::ExclusiveSum(tmp, tb, nmulti, moff, (int)rows, h->stream));
    SMLP_CK(h, cub::DeviceScan::ExclusiveSum(tmp, tb, nslot, slotoff, (int)rows, h->stream));
    totals_kernel<<<1, 1, 0, h->stream>>>(nseg, segoff, nmulti, moff, nslot, slotoff, rows, totals3);
    SMLP_CK_LAUNCH(h, "totals_kernel");
    int32_t host3[3];
    SMLP_CK(h, cudaMemcpyAsync(host3, totals3, sizeof(host3), cudaMemcpyDeviceToHost, h->stream));
    SMLP_CK(h, cudaStreamSynchronize(h->stream));
    if (host3[0] > seg_cap || host3[2] > slot_cap) {
        tmp_free(h, tmp, tb);
        tmp_free(h, buf, sizeof(int32_t) * 6 * (size_t)rows);
        return set_err(h, SMLP_E_SHAPE, "segment capacity exceeded (internal)");
    }
    seg_fill_kernel<<<grid, TPB, 0, h->stream>>>(ptr, rows, nseg, segoff, moff, slotoff, seg, multi);
    SMLP_CK_LAUNCH(h, "seg_fill_kernel");
    tmp_free(h, tmp, tb);
    tmp_free(h, buf, sizeof(int32_t) * 6 * (size_t)rows);
    return SMLP_OK;
}

}  // namespace

InitParams init_params(const smlp_handle* h, const Layer& L) {
    InitParams p{};
    p.scheme = h->init;
    const double nin = (double)L.n_in, nout = (double)L.n_out;
    if (h->init == SMLP_INIT_HE_U) p.lim = (float)std::sqrt(6.0 / nin);
    if (h->init == SMLP_INIT_XAVIER_U) p.lim = (float)std::sqrt(6.0 / (nin + nout));
    p.std = std::sqrt(2.0 / nin);
    return p;
}

int rebuild_derived(smlp_handle* h, Layer& L) {
    const int64_t nnz = L.nnz;
    // rowid
    if (nnz > 0) {
        rowid_kernel<<<launch_grid(h, nnz, TPB), TPB, 0, h->stream>>>(L.row_ptr, L.n_in, nnz, L.rowid);
        SMLP_CK_LAUNCH(h, "rowid_kernel");
    }
    // mirror: stable radix sort of (col, canonical index)
    if (nnz > 0) {
        const size_t n = (size_t)nnz;
        int32_t* buf = (int32_t*)tmp_alloc(h, sizeof(int32_t) * 3 * n);
        if (!buf) return set_err(h, SMLP_E_NOMEM, "mirror workspace");
        int32_t *idx_in = buf, *keys_out = buf + n, *dummy = buf + 2 * n;
        (void)dummy;
        iota_kernel<<<launch_grid(h, nnz, TPB), TPB, 0, h->stream>>>(idx_in, nnz);
        SMLP_CK_LAUNCH(h, "iota_kernel");
        size_t tb = 0;
        const int endbit = bits_for((uint64_t)L.n_out);
        const uint32_t* ukeys = reinterpret_cast<const uint32_t*>(L.col);
        uint32_t* ukeys_out = reinterpret_cast<uint32_t*>(keys_out);
        cub::DeviceRadixSort::SortPairs(nullptr, tb, ukeys, ukeys_out, idx_in, L.mperm, (int64_t)nnz, 0, endbit,
                                        h->stream);
        void* tmp = tmp_alloc(h, tb);
        if (!tmp) return set_err(h, SMLP_E_NOMEM, "radix temp");
        SMLP_CK(h, cub::DeviceRadixSort::SortPairs(tmp, tb, ukeys, ukeys_out, idx_in, L.mperm, (int64_t)nnz, 0,
                                                   endbit, h->stream));
        mirror_fill_kernel<<<launch_grid(h, nnz, TPB), TPB, 0, h->stream>>>(L.mperm, L.rowid, L.val, nnz, L.msrc,
                                                                             L.minv, L.mval);
        SMLP_CK_LAUNCH(h, "mirror_fill_kernel");
        mrow_ptr_kernel<<<launch_grid(h, L.n_out + 1, TPB), TPB, 0, h->stream>>>(keys_out, nnz, L.n_out, L.mrow_ptr);
        SMLP_CK_LAUNCH(h, "mrow_ptr_kernel");
        tmp_free(h, tmp, tb);
        tmp_free(h, buf, sizeof(int32_t) * 3 * n);
    } else {
        SMLP_CK(h, cudaMemsetAsync(L.mrow_ptr, 0, sizeof(int32_t) * (size_t)(L.n_out + 1), h->stream));
    }
    // segment work lists
    int32_t* tot = (int32_t*)tmp_alloc(h, sizeof(int32_t) * 8);
    if (!tot) return set_err(h, SMLP_E_NOMEM, "totals");
    SMLP_TRY(build_segments(h, L.mrow_ptr, L.n_out, L.fseg, L.fseg_cap, L.fmulti, L.fslot_cap, tot));
    SMLP_TRY(build_segments(h, L.row_ptr, L.n_in, L.bseg, L.bseg_cap, L.bmulti, L.bslot_cap, tot + 4));
    set_meta_kernel<<<1, 1, 0, h->stream>>>(L.meta, (int32_t)nnz, tot, tot + 4);
    SMLP_CK_LAUNCH(h, "set_meta_kernel");
    SMLP_CK(h, cudaMemcpyAsync(&L.meta_h, L.meta, sizeof(LayerMeta), cudaMemcpyDeviceToHost, h->stream));
    SMLP_CK(h, cudaStreamSynchronize(h->stream));
    tmp_free(h, tot, sizeof(int32_t) * 8);
    return SMLP_OK;
}

int zero_tail(smlp_handle* h, Layer& L, int64_t n) {
    if (n >= L.cap) return SMLP_OK;
    const size_t tail = (size_t)(L.cap - n);
    SMLP_CK(h, cudaMemsetAsync(L.val + n, 0, sizeof(float) * tail, h->stream));
    SMLP_CK(h, cudaMemsetAsync(L.mom + n, 0, sizeof(float) * tail, h->stream));
    SMLP_CK(h, cudaMemsetAsync(L.grad + n, 0, sizeof(float) * tail, h->stream));
    // the fused path's second gradient buffer is read by the Eq. 1 pass over the whole slice
    if (h->grad2) SMLP_CK(h, cudaMemsetAsync(h->grad2 + L.val_off + n, 0, sizeof(float) * tail, h->stream));
    return SMLP_OK;
}

int csr_from_sorted_positions(smlp_handle* h, Layer& L, const uint64_t* pos, const float* v, int64_t n) {
    SMLP_TRY(zero_tail(h, L, n));
    if (n > 0) {
        csr_from_pos_kernel<<<launch_grid(h, n, TPB), TPB, 0, h->stream>>>(pos, v, n, L.n_in, L.n_out, L.col, L.val,
                                                                            L.mom);
        SMLP_CK_LAUNCH(h, "csr_from_pos_kernel");
    }
    row_ptr_from_pos_kernel<<<launch_grid(h, L.n_in + 1, TPB), TPB, 0, h->stream>>>(pos, n, L.n_in, L.n_out,
                                                                                      L.row_ptr);
    SMLP_CK_LAUNCH(h, "row_ptr_from_pos_kernel");
    L.nnz = n;
    return rebuild_derived(h, L);
}

int fill_dense_layer(smlp_handle* h, Layer& L) {
    const InitParams ip = init_params(h, L);
    const int64_t total = L.n_in * L.n_out;
    dense_fill_kernel<<<launch_grid(h, total, TPB), TPB, 0, h->stream>>>(h->seed, (uint32_t)L.l, L.n_in, L.n_out, ip,
                                                                          L.row_ptr, L.col, L.val, L.mom);
    SMLP_CK_LAUNCH(h, "dense_fill_kernel");
    L.nnz = total;
    return rebuild_derived(h, L);
}

int first_distinct_candidates(smlp_handle* h, const Layer& L, uint32_t purpose, uint32_t c3, int64_t R,
                              bool exclude_support, const uint8_t* alive_in, const uint8_t* alive_out,
                              int64_t n_free, uint64_t* out_pos, float* out_val) {
    if (R <= 0) return SMLP_OK;
    const uint64_t n_pos = (uint64_t)L.n_in * (uint64_t)L.n_out;
    const uint64_t sentinel = n_pos;                    // sorts after every valid position
    const int endbit = bits_for(sentinel);
    const double frac = std::max(1e-9, (double)std::max<int64_t>(n_free, 1) / (double)n_pos);
    int64_t C = (int64_t)((double)R / frac * 1.25) + 1024;
    const InitParams ip = init_params(h, L);
    for (int attempt = 0; attempt < 40; ++attempt) {
        if (C > ((int64_t)1 << 31) - 1) C = ((int64_t)1 << 31) - 1;
        const size_t n = (size_t)C;
        // workspace: keys in/out (u64), m in/out (u32), flags (u8 x 3), rank (i32)
        const size_t bytes = n * (8 + 8 + 4 + 4 + 4 + 4 + 1 + 1) + 256;
        char* ws = (char*)tmp_alloc(h, bytes);
        if (!ws) return set_err(h, SMLP_E_NOMEM, "candidate workspace");
        uint64_t* keys = (uint64_t*)ws;
        uint64_t* keys_s = keys + n;
        uint32_t* ms = (uint32_t*)(keys_s + n);
        uint32_t* ms_s = ms + n;
        int32_t* rank = (int32_t*)(ms_s + n);
        int32_t* first_by_m = rank + n;
        uint8_t* first_sorted = (uint8_t*)(first_by_m + n);
        uint8_t* sel = first_sorted + n;
        const int grid = launch_grid(h, C, TPB);
        gen_candidates_kernel<<<grid, TPB, 0, h->stream>>>(h->seed, purpose, (uint32_t)L.l, c3, C, L.n_in, L.n_out,
                                                            sentinel, exclude_support, L.row_ptr, L.col, alive_in,
                                                            alive_out, keys, ms);
        SMLP_CK_LAUNCH(h, "gen_candidates_kernel");
        size_t tb = 0, tb2 = 0, tb3 = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, keys_s, ms, ms_s, C, 0, endbit, h->stream);
        cub::DeviceScan::ExclusiveSum(nullptr, tb2, first_by_m, rank, C, h->stream);
        int64_t* nsel = nullptr;
        cub::DeviceSelect::Flagged(nullptr, tb3, keys_s, sel, out_pos, nsel, C, h->stream);
        const size_t tbm = (std::max(tb, std::max(tb2, tb3)) + 255) / 256 * 256;   // keep nsel 8-aligned
        char* tmp = (char*)tmp_alloc(h, tbm + 64);
        if (!tmp) return set_err(h, SMLP_E_NOMEM, "cub temp");
        nsel = (int64_t*)(tmp + tbm);
        SMLP_CK(h, cub::DeviceRadixSort::SortPairs(tmp, tb, keys, keys_s, ms, ms_s, C, 0, endbit, h->stream));
        flag_first_kernel<<<grid, TPB, 0, h->stream>>>(keys_s, ms_s, C, sentinel, first_by_m, first_sorted);
        SMLP_CK_LAUNCH(h, "flag_first_kernel");
        SMLP_CK(h, cub::DeviceScan::ExclusiveSum(tmp, tb2, first_by_m, rank, C, h->stream));
        // distinct count D = rank[C-1] + first_by_m[C-1]
        int32_t last_rank = 0;
        int32_t last_flag = 0;
        SMLP_CK(h, cudaMemcpyAsync(&last_rank, rank + (C - 1), 4, cudaMemcpyDeviceToHost, h->stream));
        SMLP_CK(h, cudaMemcpyAsync(&last_flag, first_by_m + (C - 1), 4, cudaMemcpyDeviceToHost, h->stream));
        SMLP_CK(h, cudaStreamSynchronize(h->stream));
        const int64_t D = (int64_t)last_rank + last_flag;
        if (D >= R) {
            select_flags_kernel<<<grid, TPB, 0, h->stream>>>(ms_s, first_sorted, rank, C, R, sel);
            SMLP_CK_LAUNCH(h, "select_flags_kernel");
            SMLP_CK(h, cub::DeviceSelect::Flagged(tmp, tb3, keys_s, sel, out_pos, nsel, C, h->stream));
            // the m of each selected entry, in the same (position) order
            uint32_t* sel_m = ms;   // reuse
            SMLP_CK(h, cub::DeviceSelect::Flagged(tmp, tb3, ms_s, sel, sel_m, nsel, C, h->stream));
            candidate_values_kernel<<<launch_grid(h, R, TPB), TPB, 0, h->stream>>>(h->seed, purpose, (uint32_t)L.l,
                                                                                    c3, sel_m, R, ip, out_val);
            SMLP_CK_LAUNCH(h, "candidate_values_kernel");
            SMLP_CK(h, cudaStreamSynchronize(h->stream));
            tmp_free(h, tmp, tbm + 64);
            tmp_free(h, ws, bytes);
            return SMLP_OK;
        }
        SMLP_CK(h, cudaStreamSynchronize(h->stream));
        tmp_free(h, tmp, tbm + 64);
        tmp_free(h, ws, bytes);
        if (C >= ((int64_t)1 << 31) - 1) break;
        C *= 2;
    }
    return set_err(h, SMLP_E_ARG, "could not find enough distinct candidates (layer too saturated)");
}

int merge_layer(smlp_handle* h, Layer& L, const uint8_t* flags, const uint64_t* add_pos, const float* add_val,
                int64_t R) {
    const int64_t nnz = L.nnz;
    int32_t* s = (int32_t*)tmp_alloc(h, sizeof(int32_t) * (size_t)(nnz + 1));
    int32_t* sp = (int32_t*)tmp_alloc(h, sizeof(int32_t) * (size_t)(nnz + 1));
    if (!s || !sp) return set_err(h, SMLP_E_NOMEM, "merge workspace");
    survivor_flags_kernel<<<launch_grid(h, nnz + 1, TPB), TPB, 0, h->stream>>>(flags, nnz, s);
    SMLP_CK_LAUNCH(h, "survivor_flags_kernel");
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, s, sp, nnz + 1, h->stream);
    void* tmp = tmp_alloc(h, tb);
    if (!tmp) return set_err(h, SMLP_E_NOMEM, "scan temp");
    SMLP_CK(h, cub::DeviceScan::ExclusiveSum(tmp, tb, s, sp, nnz + 1, h->stream));
    int32_t n_surv = 0;
    SMLP_CK(h, cudaMemcpyAsync(&n_surv, sp + nnz, 4, cudaMemcpyDeviceToHost, h->stream));
    SMLP_CK(h, cudaStreamSynchronize(h->stream));
    const int64_t new_nnz = (int64_t)n_surv + R;
    if (new_nnz > L.cap) return set_err(h, SMLP_E_SHAPE, "layer capacity exceeded");
    const size_t nb = (size_t)std::max<int64_t>(new_nnz, 1);
    int32_t* ncol = (int32_t*)tmp_alloc(h, sizeof(int32_t) * nb);
    float* nval = (float*)tmp_alloc(h, sizeof(float) * nb);
    float* nmom = (float*)tmp_alloc(h, sizeof(float) * nb);
    int32_t* nrp = (int32_t*)tmp_alloc(h, sizeof(int32_t) * (size_t)(L.n_in + 1));
    if (!ncol || !nval || !nmom || !nrp) return set_err(h, SMLP_E_NOMEM, "merge buffers");
    if (nnz > 0) {
        merge_survivors_kernel<<<launch_grid(h, nnz, TPB), TPB, 0, h->stream>>>(
            L.rowid, L.col, L.val, L.mom, flags, sp, add_pos, R, nnz, L.n_out, ncol, nval, nmom);
        SMLP_CK_LAUNCH(h, "merge_survivors_kernel");
    }
    if (R > 0) {
        merge_additions_kernel<<<launch_grid(h, R, TPB), TPB, 0, h->stream>>>(L.row_ptr, L.col, sp, add_pos, add_val,
                                                                               R, L.n_out, ncol, nval, nmom);
        SMLP_CK_LAUNCH(h, "merge_additions_kernel");
    }
    merge_row_ptr_kernel<<<launch_grid(h, L.n_in + 1, TPB), TPB, 0, h->stream>>>(L.row_ptr, sp, add_pos, R, L.n_in,
                                                                                   L.n_out, nrp);
    SMLP_CK_LAUNCH(h, "merge_row_ptr_kernel");
    // copy back into the graph-stable buffers; the tail beyond new_nnz is zeroed so the param /
    // grad views stay clean after pruning
    SMLP_CK(h, cudaMemcpyAsync(L.col, ncol, sizeof(int32_t) * (size_t)new_nnz, cudaMemcpyDeviceToDevice, h->stream));
    SMLP_CK(h, cudaMemcpyAsync(L.val, nval, sizeof(float) * (size_t)new_nnz, cudaMemcpyDeviceToDevice, h->stream));
    SMLP_CK(h, cudaMemcpyAsync(L.mom, nmom, sizeof(float) * (size_t)new_nnz, cudaMemcpyDeviceToDevice, h->stream));
    SMLP_CK(h, cudaMemcpyAsync(L.row_ptr, nrp, sizeof(int32_t) * (size_t)(L.n_in + 1), cudaMemcpyDeviceToDevice,
                               h->stream));
    SMLP_TRY(zero_tail(h, L, new_nnz));
    SMLP_CK(h, cudaStreamSynchronize(h->stream));
    tmp_free(h, ncol, sizeof(int32_t) * nb);
    tmp_free(h, nval, sizeof(float) * nb);
    tmp_free(h, nmom, sizeof(float) * nb);
    tmp_free(h, nrp, sizeof(int32_t) * (size_t)(L.n_in + 1));
    tmp_free(h, tmp, tb);
    tmp_free(h, s, sizeof(int32_t) * (size_t)(nnz + 1));
    tmp_free(h, sp, sizeof(int32_t) * (size_t)(nnz + 1));
    L.nnz = new_nnz;
    return rebuild_derived(h, L);
}

int compact_layer(smlp_handle* h, Layer& L, const uint8_t* remove_flags) {
    return merge_layer(h, L, remove_flags, nullptr, nullptr, 0);
}

}  // namespace smlp
