// step.cu — the per-minibatch hot path on sm_100a CUDA cores.
//
//   stage_input    a1  x[B x n_1] (optionally row-gathered by x_idx) -> act[1] chunked transposed
//   fwd_kernel     a2/a3  z_l = a_{l-1} W^(l) + b_l over the output-major mirror.  A "group" of
//                  G = CB/4 lanes owns one <= SEG_NNZ-entry segment of an output row (P = 32/G groups
//                  per warp run in lock-step, predicated to the longest segment); each lane holds one
//                  float4 of the CB batch columns; per block of G entries the group loads (src, w)
//                  coalesced, broadcasts them by shuffle, and keeps G row gathers in flight (the next
//                  block's indices are prefetched).  Epilogue: bias, All-ReLU (Eq. 3),
//                  inverted dropout (Philox), sign / keep bit masks.
//   fwd_finish     rows split into several segments: fixed-order sum of the partials + epilogue
//   softmax_ce     a3  p = softmax(z_L), loss, delta_L = (p - onehot)/B, output-bias gradient
//   bwd_kernel     a4/a5/a6  a group owns a segment of an input row i of the canonical CSR: per
//                  entry it gathers delta_l[j] once, accumulates delta_{l-1}[i] += w_ij delta_l[j]
//                  (SpMM against W^T) and the partial dot <a_{l-1}[i], delta_l[j]> (SDDMM); a
//                  transpose reduction over the G lanes leaves lane q with the batch sum of entry q,
//                  which it applies as the Eq. 1 update of (w, v) in place (1-GPU fused path, also
//                  refreshing the forward's mirror-ordered copy of w) or writes to the grad view
//   bwd_finish     multi-segment rows: fixed-order sum of the delta partials + epilogue
//   sgd_update     a6 on the grad view after the caller's allreduce (K > 1), then mirror refresh
//
// Batch chunks: with CB < B the batch is processed in ceil(B/CB) chunk launches so the gathered
// activation slab (n x CB fp32) stays L2-resident; gradients accumulate over chunks in order.
// No float atomics anywhere: every reduction has a fixed order, so results are deterministic.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "smlp_internal.cuh"

namespace smlp {
namespace {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ float4 ldg4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
__device__ __forceinline__ float4 f4zero() { return make_float4(0.f, 0.f, 0.f, 0.f); }
__device__ __forceinline__ void fma4(float4& acc, float w, const float4& x) {
    acc.x = fmaf(w, x.x, acc.x);
    acc.y = fmaf(w, x.y, acc.y);
    acc.z = fmaf(w, x.z, acc.z);
    acc.w = fmaf(w, x.w, acc.w);
}
__device__ __forceinline__ float comp(const float4& v, int c) {
    return c == 0 ? v.x : (c == 1 ? v.y : (c == 2 ? v.z : v.w));
}
__device__ __forceinline__ uint32_t word(const uint4& v, int c) {
    return c == 0 ? v.x : (c == 1 ? v.y : (c == 2 ? v.z : v.w));
}
template <int G>
__device__ __forceinline__ uint32_t group_bits(uint32_t ballot, int g) {
    return G == 32 ? ballot : ((ballot >> (g * G)) & ((1u << G) - 1u));
}

// ------------------------------------------------------------------------------------------
// a1: input staging (transpose + optional row gather), zero padding of columns b >= B
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) stage_input_kernel(const float* __restrict__ x, const int32_t* __restrict__ x_idx,
                                                           int B, int nchunks, int CB, int64_t n1,
                                                           float* __restrict__ act1) {
    __shared__ float tile[32][33];
    const int64_t f0 = (int64_t)blockIdx.x * 32;
    const int b0 = blockIdx.y * 32;
    const int tx = threadIdx.x, ty = threadIdx.y;   // 32 x 32
    {
        const int b = b0 + ty;
        const int64_t f = f0 + tx;
        float v = 0.f;
        if (b < B && f < n1) {
            const int64_t row = x_idx ? (int64_t)__ldg(x_idx + b) : (int64_t)b;
            v = __ldg(x + row * n1 + f);
        }
        tile[ty][tx] = v;
    }
    __syncthreads();
    {
        const int b = b0 + tx;
        const int64_t f = f0 + ty;
        if (f < n1 && b < nchunks * CB) {
            const int c = b / CB, lb = b % CB;
            act1[((int64_t)c * n1 + f) * CB + lb] = tile[tx][ty];
        }
    }
}

// ------------------------------------------------------------------------------------------
// forward
// ------------------------------------------------------------------------------------------
struct FwdArgs {
    const float* a_prev;      // chunk base [n_in][CB]
    float* a_out;             // chunk base [n_out][CB]
    uint4* zmask;             // chunk base [n_out] (hidden layers)
    uint4* kmask;             // chunk base [n_out] (hidden layers with dropout)
    const int4* seg;
    const int4* multi;
    const LayerMeta* meta;
    const int32_t* msrc;      // mirror: input neuron of each entry
    const float* mval;        // mirror-ordered copy of the weights
    const float* bias;
    float* ws;
    int64_t n_out;
    int hidden;               // 1: All-ReLU/ReLU + dropout epilogue; 0: output logits
    float neg_slope;          // slope of f_l for z <= 0
    int dropout_on;
    uint32_t drop_thr;        // keep iff word >= floor(rate 2^32)
    float keep_scale;         // 1/(1-rate)
    uint64_t seed;
    int rank;
    int layer;
    uint32_t step_lo;
    const uint64_t* step_ptr; // device dropout-step source (graph replay) or null
    int b0;                   // global batch index of column 0 of this chunk
};

// Epilogue of one output row j per group: all 32 lanes call it (ballots); `own` marks the
// groups whose row is complete here.  Lane q of a group owns batch columns 4q..4q+3 of the chunk.
template <int CB>
__device__ __forceinline__ void fwd_epilogue(const FwdArgs& A, int64_t j, float4 acc, bool own, int lane,
                                             uint32_t step_lo) {
    constexpr int G = CB / 4;
    const int g = lane / G, q = lane % G;
    const float bj = own ? __ldg(A.bias + j) : 0.f;
    const float4 z = make_float4(acc.x + bj, acc.y + bj, acc.z + bj, acc.w + bj);
    if (!A.hidden) {
        if (own) st4(A.a_out + j * CB + q * 4, z);
        return;
    }
    uint32_t zb[4], kb[4];
    float out[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const float zc = comp(z, c);
        const bool pos = zc > 0.f;
        zb[c] = group_bits<G>(__ballot_sync(FULL, own && pos), g);
        float a = pos ? zc : A.neg_slope * zc;
        bool keep = true;
        if (A.dropout_on) {
            const uint64_t b = (uint64_t)(A.b0 + q * 4 + c);
            const uint64_t e = b * (uint64_t)A.n_out + (uint64_t)j;
            const uint4 r = rng_stream(A.seed, P_DROPOUT, A.rank, A.layer, step_lo, e >> 2);
            keep = word(r, (int)(e & 3)) >= A.drop_thr;
            a = keep ? a * A.keep_scale : 0.f;
        }
        kb[c] = group_bits<G>(__ballot_sync(FULL, own && keep), g);
        out[c] = a;
    }
    if (own) {
        st4(A.a_out + j * CB + q * 4, make_float4(out[0], out[1], out[2], out[3]));
        if (q == 0) {
            A.zmask[j] = make_uint4(zb[0], zb[1], zb[2], zb[3]);
            if (A.dropout_on) A.kmask[j] = make_uint4(kb[0], kb[1], kb[2], kb[3]);
        }
    }
}

// Gather-accumulate of one segment [beg, end) per group (groups in lock-step up to maxblk).
template <int CB>
__device__ __forceinline__ float4 fwd_segment(const FwdArgs& A, int beg, int end, int maxblk, int lane) {
    constexpr int G = CB / 4;
    constexpr int U = G < 8 ? G : 8;
    const int g = lane / G, q = lane % G, gbase = g * G;
    float4 acc = f4zero();
    int k = beg + q;
    int src = 0;
    float w = 0.f;
    if (k < end) {
        src = __ldg(A.msrc + k);
        w = __ldg(A.mval + k);
    }
    for (int b = 0; b < maxblk; ++b) {
        const int kn = k + G;                          // prefetch the next block's entries
        int src_n = 0;
        float w_n = 0.f;
        if (kn < end) {
            src_n = __ldg(A.msrc + kn);
            w_n = __ldg(A.mval + kn);
        }
        const int base = beg + b * G;
#pragma unroll
        for (int u0 = 0; u0 < G; u0 += U) {
            float4 x[U];
            float wv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int s = __shfl_sync(FULL, src, gbase + u0 + u);
                wv[u] = __shfl_sync(FULL, w, gbase + u0 + u);
                x[u] = (base + u0 + u < end) ? ldg4(A.a_prev + (int64_t)s * CB + q * 4) : f4zero();
            }
#pragma unroll
            for (int u = 0; u < U; ++u) fma4(acc, wv[u], x[u]);
        }
        k = kn;
        src = src_n;
        w = w_n;
    }
    return acc;
}

template <int CB>
__global__ void __launch_bounds__(256) fwd_kernel(FwdArgs A) {
    constexpr int G = CB / 4, P = 32 / G;
    const int lane = threadIdx.x & 31, g = lane / G, q = lane % G;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    const int nseg = A.meta->n_fseg;
    const uint32_t step_lo = A.step_ptr ? (uint32_t)(*A.step_ptr) : A.step_lo;
    for (int s0 = warp * P; s0 < nseg; s0 += nwarps * P) {
        const int s = s0 + g;
        const bool active = s < nseg;
        const int4 sg = active ? A.seg[s] : make_int4(0, 0, 0, -2);
        const int nblk = (sg.z - sg.y + G - 1) / G;
        const int maxblk = __reduce_max_sync(FULL, nblk);
        const float4 acc = fwd_segment<CB>(A, sg.y, sg.z, maxblk, lane);
        fwd_epilogue<CB>(A, sg.x, acc, active && sg.w < 0, lane, step_lo);
        if (active && sg.w >= 0) st4(A.ws + (int64_t)sg.w * CB + q * 4, acc);
    }
}

template <int CB>
__global__ void __launch_bounds__(256) fwd_finish_kernel(FwdArgs A) {
    constexpr int G = CB / 4, P = 32 / G;
    const int lane = threadIdx.x & 31, g = lane / G, q = lane % G;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    const int nm = A.meta->n_fmulti;
    const uint32_t step_lo = A.step_ptr ? (uint32_t)(*A.step_ptr) : A.step_lo;
    for (int r0 = warp * P; r0 < nm; r0 += nwarps * P) {
        const int r = r0 + g;
        const bool active = r < nm;
        const int4 m = active ? A.multi[r] : make_int4(0, 0, 0, 0);
        float4 acc = f4zero();
        for (int t = 0; t < m.z; ++t) {          // fixed order: slot first .. first + n - 1
            const float4 p = ldg4(A.ws + (int64_t)(m.y + t) * CB + q * 4);
            acc.x += p.x; acc.y += p.y; acc.z += p.z; acc.w += p.w;
        }
        fwd_epilogue<CB>(A, m.x, acc, active, lane, step_lo);
    }
}

// ------------------------------------------------------------------------------------------
// softmax cross-entropy (single block, fixed-order reductions)
// ------------------------------------------------------------------------------------------
struct SoftmaxArgs {
    const float* logits;      // act[L] [nchunks][n_L][CB]
    float* delta;             // delta[L] same layout
    const int32_t* labels;
    const int32_t* y_idx;
    float* loss;              // scalar or null
    int32_t* err;
    float* bias;              // b_L
    float* bias_mom;
    float* bias_grad;         // grad view slice (unfused)
    int64_t nL;
    int B, nchunks, CB;
    int fused;
    float lr, mu;
};

__global__ void __launch_bounds__(512) softmax_ce_kernel(SoftmaxArgs A) {
    __shared__ double red[512];
    const int tid = threadIdx.x;
    double lsum = 0.0;
    const int total = A.nchunks * A.CB;
    const float invB = 1.0f / (float)A.B;
    for (int b = tid; b < total; b += blockDim.x) {
        const int c = b / A.CB, lb = b % A.CB;
        const float* zc = A.logits + (int64_t)c * A.nL * A.CB + lb;
        float* dc = A.delta + (int64_t)c * A.nL * A.CB + lb;
        if (b >= A.B) {
            for (int64_t j = 0; j < A.nL; ++j) dc[j * A.CB] = 0.f;
            continue;
        }
        int y = A.labels[A.y_idx ? A.y_idx[b] : b];
        if (y < 0 || y >= A.nL) {
            atomicOr(A.err, 1);
            y = 0;
        }
        float mx = -INFINITY;
        for (int64_t j = 0; j < A.nL; ++j) mx = fmaxf(mx, zc[j * A.CB]);
        float s = 0.f;
        for (int64_t j = 0; j < A.nL; ++j) s += expf(zc[j * A.CB] - mx);
        const float lse = logf(s);
        lsum += (double)(lse - (zc[(int64_t)y * A.CB] - mx));
        const float inv = 1.0f / s;
        for (int64_t j = 0; j < A.nL; ++j) {
            const float p = expf(zc[j * A.CB] - mx) * inv;
            dc[j * A.CB] = (p - (j == y ? 1.f : 0.f)) * invB;
        }
    }
    red[tid] = lsum;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (tid < s) red[tid] += red[tid + s];
        __syncthreads();
    }
    if (tid == 0 && A.loss) *A.loss = (float)(red[0] / (double)A.B);
    // output-layer bias gradient gb_L = sum_b delta_L[b, :]
    for (int64_t j = tid; j < A.nL; j += blockDim.x) {
        float g = 0.f;
        for (int c = 0; c < A.nchunks; ++c) {
            const float* dc = A.delta + ((int64_t)c * A.nL + j) * A.CB;
            for (int lb = 0; lb < A.CB; ++lb) g += dc[lb];
        }
        if (A.fused) {
            const float v = A.mu * A.bias_mom[j] - A.lr * g;
            A.bias_mom[j] = v;
            A.bias[j] = A.bias[j] + v;
        } else {
            A.bias_grad[j] = g;
        }
    }
}

__global__ void softmax_probs_kernel(const float* __restrict__ logits, float* __restrict__ probs, int64_t nL, int B,
                                     int CB) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    const int c = b / CB, lb = b % CB;
    const float* zc = logits + (int64_t)c * nL * CB + lb;
    float mx = -INFINITY;
    for (int64_t j = 0; j < nL; ++j) mx = fmaxf(mx, zc[j * CB]);
    float s = 0.f;
    for (int64_t j = 0; j < nL; ++j) s += expf(zc[j * CB] - mx);
    const float inv = 1.0f / s;
    for (int64_t j = 0; j < nL; ++j) probs[(int64_t)b * nL + j] = expf(zc[j * CB] - mx) * inv;
}

// ------------------------------------------------------------------------------------------
// backward (delta SpMM against W^T + SDDMM + fused update)
// ------------------------------------------------------------------------------------------
struct BwdArgs {
    const float* a_prev;      // chunk base [n_in][CB]   (activations of layer l-1)
    const float* d_out;       // chunk base [n_out][CB]  (delta_l)
    float* d_prev;            // chunk base [n_in][CB]   (delta_{l-1}) or null for l = 2
    const uint4* zmask_prev;  // chunk base [n_in]
    const uint4* kmask_prev;
    const int4* seg;
    const int4* multi;
    const LayerMeta* meta;
    const int32_t* col;
    float* val;
    float* mom;
    float* grad;
    float* mval;              // mirror-ordered copy of w (refreshed by the fused update)
    const int32_t* minv;      // canonical index -> mirror position
    float* ws;
    float* bgs;               // [n_in] bias-grad accumulator over chunks
    float* bias_prev;
    float* bias_mom_prev;
    float* bias_grad_prev;
    float neg_slope_prev;
    float keep_scale_prev;
    int dropout_prev;
    int chunk, nchunks;
    int fused;
    float lr, mu, wd;
};

// delta_{l-1} of input row i per group: f'(z) from the sign bits, dropout keep bits, store, and
// the bias gradient of layer l-1 (accumulated across chunks in order).
template <int CB>
__device__ __forceinline__ void bwd_epilogue(const BwdArgs& A, int64_t i, float4 d, bool own, int lane) {
    constexpr int G = CB / 4;
    const int q = lane % G;
    float o[4] = {0.f, 0.f, 0.f, 0.f};
    if (own) {
        const uint4 zb = A.zmask_prev[i];
        uint4 kb = make_uint4(FULL, FULL, FULL, FULL);
        if (A.dropout_prev) kb = A.kmask_prev[i];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const bool pos = (word(zb, c) >> q) & 1u;
            const bool keep = (word(kb, c) >> q) & 1u;
            const float fp = pos ? 1.f : A.neg_slope_prev;
            const float v = comp(d, c) * fp;
            o[c] = A.dropout_prev ? (keep ? v * A.keep_scale_prev : 0.f) : v;
        }
        st4(A.d_prev + i * CB + q * 4, make_float4(o[0], o[1], o[2], o[3]));
    }
    float s = (o[0] + o[1]) + (o[2] + o[3]);
#pragma unroll
    for (int m = 1; m < G; m <<= 1) s += __shfl_xor_sync(FULL, s, m);
    if (own && q == 0) {
        float tot = s;
        if (A.chunk > 0) tot += A.bgs[i];
        if (A.chunk + 1 < A.nchunks) {
            A.bgs[i] = tot;
        } else if (A.fused) {
            const float v = A.mu * A.bias_mom_prev[i] - A.lr * tot;
            A.bias_mom_prev[i] = v;
            A.bias_prev[i] = A.bias_prev[i] + v;
        } else {
            A.bias_grad_prev[i] = tot;
        }
    }
}

template <int CB, bool HAS_DPREV>
__global__ void __launch_bounds__(256) bwd_kernel(BwdArgs A) {
    constexpr int G = CB / 4, P = 32 / G;
    constexpr int U = G < 8 ? G : 8;
    const int lane = threadIdx.x & 31;
    const int g = lane / G, q = lane % G, gbase = g * G;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    const int nseg = A.meta->n_bseg;
    const bool first_chunk = A.chunk == 0, last_chunk = A.chunk + 1 == A.nchunks;
    for (int s0 = warp * P; s0 < nseg; s0 += nwarps * P) {
        const int s = s0 + g;
        const bool active = s < nseg;
        const int4 sg = active ? A.seg[s] : make_int4(0, 0, 0, -2);
        const int64_t i = sg.x;
        const int beg = sg.y, end = sg.z;
        const int maxblk = __reduce_max_sync(FULL, (end - beg + G - 1) / G);
        const float4 ai = active ? ldg4(A.a_prev + i * CB + q * 4) : f4zero();
        float4 dacc = f4zero();
        int k = beg + q;
        int jcol = 0;
        float w = 0.f;
        if (k < end) {
            jcol = __ldg(A.col + k);
            w = A.val[k];
        }
        for (int b = 0; b < maxblk; ++b) {
            const int kn = k + G;                      // prefetch the next block's entries
            int jcol_n = 0;
            float w_n = 0.f;
            if (kn < end) {
                jcol_n = __ldg(A.col + kn);
                w_n = A.val[kn];
            }
            const int base = beg + b * G;
            float p[G];
#pragma unroll
            for (int u0 = 0; u0 < G; u0 += U) {
                float4 dx[U];
                float wv[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int jj = __shfl_sync(FULL, jcol, gbase + u0 + u);
                    wv[u] = __shfl_sync(FULL, w, gbase + u0 + u);
                    dx[u] = (base + u0 + u < end) ? ldg4(A.d_out + (int64_t)jj * CB + q * 4) : f4zero();
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if (HAS_DPREV) fma4(dacc, wv[u], dx[u]);
                    p[u0 + u] = fmaf(ai.x, dx[u].x, fmaf(ai.y, dx[u].y, fmaf(ai.z, dx[u].z, ai.w * dx[u].w)));
                }
            }
            // transpose reduction over the G lanes of the group: lane q ends with the batch sum
            // of entry q of this block (= its own entry k)
#pragma unroll
            for (int h = G / 2; h >= 1; h >>= 1) {
                const bool upper = (q & h) != 0;
#pragma unroll
                for (int u = 0; u < h; ++u) {
                    const float send = upper ? p[u] : p[u + h];
                    const float keep = upper ? p[u + h] : p[u];
                    p[u] = keep + __shfl_xor_sync(FULL, send, h);
                }
            }
            if (k < end) {
                float gk = p[0];
                if (!first_chunk) gk += A.grad[k];
                if (!last_chunk || !A.fused) {
                    A.grad[k] = gk;
                } else {
                    const float v = A.mu * A.mom[k] - A.lr * (gk + A.wd * w);
                    const float wn = w + v;
                    A.mom[k] = v;
                    A.val[k] = wn;
                    A.mval[__ldg(A.minv + k)] = wn;
                }
            }
            k = kn;
            jcol = jcol_n;
            w = w_n;
        }
        if (HAS_DPREV) {
            bwd_epilogue<CB>(A, i, dacc, active && sg.w < 0, lane);
            if (active && sg.w >= 0) st4(A.ws + (int64_t)sg.w * CB + q * 4, dacc);
        }
    }
}

template <int CB>
__global__ void __launch_bounds__(256) bwd_finish_kernel(BwdArgs A) {
    constexpr int G = CB / 4, P = 32 / G;
    const int lane = threadIdx.x & 31, g = lane / G, q = lane % G;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    const int nm = A.meta->n_bmulti;
    for (int r0 = warp * P; r0 < nm; r0 += nwarps * P) {
        const int r = r0 + g;
        const bool active = r < nm;
        const int4 m = active ? A.multi[r] : make_int4(0, 0, 0, 0);
        float4 acc = f4zero();
        for (int t = 0; t < m.z; ++t) {
            const float4 p = ldg4(A.ws + (int64_t)(m.y + t) * CB + q * 4);
            acc.x += p.x; acc.y += p.y; acc.z += p.z; acc.w += p.w;
        }
        bwd_epilogue<CB>(A, m.x, acc, active, lane);
    }
}

// ------------------------------------------------------------------------------------------
// a6 standalone: Eq. 1 over the whole grad view (K > 1 path), then the mirror refresh
// ------------------------------------------------------------------------------------------
__global__ void sgd_update_kernel(float* __restrict__ w, float* __restrict__ v, const float* __restrict__ g,
                                  int64_t n, int64_t bias_base, float lr, float mu, float wd, float gs) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        const float wk = w[k];
        const float lam = k < bias_base ? wd : 0.f;
        const float vk = mu * v[k] - lr * (gs * g[k] + lam * wk);
        v[k] = vk;
        w[k] = wk + vk;
    }
}

__global__ void mirror_values_kernel(const float* __restrict__ val, const int32_t* __restrict__ mperm,
                                     const LayerMeta* __restrict__ meta, float* __restrict__ mval) {
    const int64_t n = meta->nnz;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
        mval[t] = __ldg(val + __ldg(mperm + t));
}

int persistent_grid(const smlp_handle* h, int64_t groups, int groups_per_warp) {
    const int64_t warps = (groups + groups_per_warp - 1) / groups_per_warp;
    const int64_t need = (warps + WARPS_PER_BLOCK - 1) / WARPS_PER_BLOCK;
    const int64_t cap = (int64_t)h->num_sms * 8;
    return (int)std::max<int64_t>(1, std::min(need, cap));
}

template <int CB>
int launch_fwd(smlp_handle* h, const FwdArgs& A, const Layer& L) {
    constexpr int P = 32 / (CB / 4);
    const int grid = persistent_grid(h, L.fseg_cap, P);
    fwd_kernel<CB><<<grid, WARPS_PER_BLOCK * 32, 0, h->stream>>>(A);
    SMLP_CK_LAUNCH(h, "fwd_kernel");
    if (L.fslot_cap > 0) {
        const int g2 = persistent_grid(h, std::max<int64_t>(1, L.fslot_cap / 2), P);
        fwd_finish_kernel<CB><<<g2, WARPS_PER_BLOCK * 32, 0, h->stream>>>(A);
        SMLP_CK_LAUNCH(h, "fwd_finish_kernel");
    }
    return SMLP_OK;
}

template <int CB>
int launch_bwd(smlp_handle* h, const BwdArgs& A, const Layer& L, bool has_dprev) {
    constexpr int P = 32 / (CB / 4);
    const int grid = persistent_grid(h, L.bseg_cap, P);
    if (has_dprev) {
        bwd_kernel<CB, true><<<grid, WARPS_PER_BLOCK * 32, 0, h->stream>>>(A);
    } else {
        bwd_kernel<CB, false><<<grid, WARPS_PER_BLOCK * 32, 0, h->stream>>>(A);
    }
    SMLP_CK_LAUNCH(h, "bwd_kernel");
    if (has_dprev && L.bslot_cap > 0) {
        const int g2 = persistent_grid(h, std::max<int64_t>(1, L.bslot_cap / 2), P);
        bwd_finish_kernel<CB><<<g2, WARPS_PER_BLOCK * 32, 0, h->stream>>>(A);
        SMLP_CK_LAUNCH(h, "bwd_finish_kernel");
    }
    return SMLP_OK;
}

#define SMLP_DISPATCH_CB(h, fn, ...)                                   \
    switch ((h)->CB) {                                                 \
        case 4: return fn<4>(__VA_ARGS__);                             \
        case 8: return fn<8>(__VA_ARGS__);                             \
        case 16: return fn<16>(__VA_ARGS__);                           \
        case 32: return fn<32>(__VA_ARGS__);                           \
        case 64: return fn<64>(__VA_ARGS__);                           \
        case 128: return fn<128>(__VA_ARGS__);                         \
        default: return set_err((h), SMLP_E_ARG, "unsupported chunk_batch"); \
    }

int dispatch_fwd(smlp_handle* h, const FwdArgs& A, const Layer& L) { SMLP_DISPATCH_CB(h, launch_fwd, h, A, L); }
int dispatch_bwd(smlp_handle* h, const BwdArgs& A, const Layer& L, bool hd) { SMLP_DISPATCH_CB(h, launch_bwd, h, A, L, hd); }

float neg_slope_of(const smlp_handle* h, int l) {
    if (h->activation == SMLP_ACT_RELU) return 0.f;
    return (l % 2 == 0) ? -h->alpha : h->alpha;   // Eq. 3: -alpha x for even l, +alpha x for odd l
}

uint32_t drop_threshold(float rate) {
    const double t = std::floor((double)rate * 4294967296.0);
    return (uint32_t)std::min(t, 4294967295.0);
}

}  // namespace

int refresh_mirror_values(smlp_handle* h, Layer& Ly) {
    if (Ly.cap == 0) return SMLP_OK;
    mirror_values_kernel<<<launch_grid(h, Ly.cap, 256), 256, 0, h->stream>>>(Ly.val, Ly.mperm, Ly.meta, Ly.mval);
    SMLP_CK_LAUNCH(h, "mirror_values_kernel");
    return SMLP_OK;
}

int run_probs(smlp_handle* h, int B, float* probs) {
    softmax_probs_kernel<<<(B + 127) / 128, 128, 0, h->stream>>>(h->act[h->L], probs, h->sizes[h->L - 1], B, h->CB);
    SMLP_CK_LAUNCH(h, "softmax_probs_kernel");
    return SMLP_OK;
}

int run_forward(smlp_handle* h, const float* x, const int32_t* x_idx, int B, bool train, uint64_t step,
                float* probs) {
    const int CB = h->CB;
    const int nchunks = (B + CB - 1) / CB;
    {
        dim3 grid((unsigned)((h->sizes[0] + 31) / 32), (unsigned)((nchunks * CB + 31) / 32));
        prof_start(h, K_STAGE, 1, 8.0 * (double)B * (double)h->sizes[0], 0.0);
        stage_input_kernel<<<grid, dim3(32, 32), 0, h->stream>>>(x, x_idx, B, nchunks, CB, h->sizes[0], h->act[1]);
        SMLP_CK_LAUNCH(h, "stage_input_kernel");
        prof_stop(h);
    }
    const bool drop = train && h->dropout > 0.f;
    for (int c = 0; c < nchunks; ++c) {
        for (int l = 2; l <= h->L; ++l) {
            Layer& Ly = h->layers[l - 2];
            const int64_t nin = h->sizes[l - 2], nout = h->sizes[l - 1];
            FwdArgs A{};
            A.a_prev = h->act[l - 1] + (int64_t)c * nin * CB;
            A.a_out = h->act[l] + (int64_t)c * nout * CB;
            const bool hidden = l < h->L;
            A.zmask = hidden ? h->zmask[l] + (int64_t)c * nout : nullptr;
            A.kmask = hidden ? h->kmask[l] + (int64_t)c * nout : nullptr;
            A.seg = Ly.fseg;
            A.multi = Ly.fmulti;
            A.meta = Ly.meta;
            A.msrc = Ly.msrc;
            A.mval = Ly.mval;
            A.bias = Ly.bias;
            A.ws = Ly.fws;
            A.n_out = nout;
            A.hidden = hidden ? 1 : 0;
            A.neg_slope = neg_slope_of(h, l);
            A.dropout_on = (hidden && drop) ? 1 : 0;
            A.drop_thr = drop_threshold(h->dropout);
            A.keep_scale = (float)(1.0 / (1.0 - (double)h->dropout));
            A.seed = h->seed;
            A.rank = h->rank;
            A.layer = l;
            A.step_lo = (uint32_t)step;
            A.step_ptr = h->step_counter;
            A.b0 = c * CB;
            const int Bc = std::min(CB, B - c * CB);
            const double nnz = (double)Ly.nnz;
            prof_start(h, K_FWD, l, 12.0 * nnz / nchunks + 4.0 * Bc * (double)(nin + nout), 2.0 * nnz * Bc);
            SMLP_TRY(dispatch_fwd(h, A, Ly));
            prof_stop(h);
        }
    }
    if (probs) SMLP_TRY(run_probs(h, B, probs));
    h->trace_valid = true;
    h->trace_train = train;
    h->trace_B = B;
    h->trace_version = h->version;
    h->trace_step = step;
    return SMLP_OK;
}

int run_backward(smlp_handle* h, const int32_t* labels, const int32_t* y_idx, float* loss, const smlp_sgd* fused) {
    const int CB = h->CB;
    const int B = h->trace_B;
    const int nchunks = (B + CB - 1) / CB;
    const int L = h->L;
    const bool is_fused = fused != nullptr;
    const float lr = is_fused ? fused->lr : 0.f, mu = is_fused ? fused->momentum : 0.f,
                wd = is_fused ? fused->weight_decay : 0.f;
    {
        Layer& Lo = h->layers[L - 2];
        SoftmaxArgs S{};
        S.logits = h->act[L];
        S.delta = h->delta[L];
        S.labels = labels;
        S.y_idx = y_idx;
        S.loss = loss;
        S.err = h->d_err;
        S.bias = Lo.bias;
        S.bias_mom = Lo.bias_mom;
        S.bias_grad = Lo.bias_grad;
        S.nL = h->sizes[L - 1];
        S.B = B;
        S.nchunks = nchunks;
        S.CB = CB;
        S.fused = is_fused ? 1 : 0;
        S.lr = lr;
        S.mu = mu;
        prof_start(h, K_SOFTMAX, L, 8.0 * (double)B * (double)S.nL, 0.0);
        softmax_ce_kernel<<<1, 512, 0, h->stream>>>(S);
        SMLP_CK_LAUNCH(h, "softmax_ce_kernel");
        prof_stop(h);
    }
    for (int l = L; l >= 2; --l) {
        Layer& Ly = h->layers[l - 2];
        const int64_t nin = h->sizes[l - 2], nout = h->sizes[l - 1];
        const bool has_dprev = l >= 3;
        Layer* Lp = has_dprev ? &h->layers[l - 3] : nullptr;   // owner of bias b_{l-1}
        for (int c = 0; c < nchunks; ++c) {
            BwdArgs A{};
            A.a_prev = h->act[l - 1] + (int64_t)c * nin * CB;
            A.d_out = h->delta[l] + (int64_t)c * nout * CB;
            A.d_prev = has_dprev ? h->delta[l - 1] + (int64_t)c * nin * CB : nullptr;
            A.zmask_prev = has_dprev ? h->zmask[l - 1] + (int64_t)c * nin : nullptr;
            A.kmask_prev = has_dprev ? h->kmask[l - 1] + (int64_t)c * nin : nullptr;
            A.seg = Ly.bseg;
            A.multi = Ly.bmulti;
            A.meta = Ly.meta;
            A.col = Ly.col;
            A.val = Ly.val;
            A.mom = Ly.mom;
            A.grad = Ly.grad;
            A.mval = Ly.mval;
            A.minv = Ly.minv;
            A.ws = Ly.bws;
            A.bgs = Ly.bgs;
            A.bias_prev = Lp ? Lp->bias : nullptr;
            A.bias_mom_prev = Lp ? Lp->bias_mom : nullptr;
            A.bias_grad_prev = Lp ? Lp->bias_grad : nullptr;
            A.neg_slope_prev = neg_slope_of(h, l - 1);
            A.dropout_prev = (has_dprev && h->trace_train && h->dropout > 0.f) ? 1 : 0;
            A.keep_scale_prev = (float)(1.0 / (1.0 - (double)h->dropout));
            A.chunk = c;
            A.nchunks = nchunks;
            A.fused = is_fused ? 1 : 0;
            A.lr = lr;
            A.mu = mu;
            A.wd = wd;
            const int Bc = std::min(CB, B - c * CB);
            const double nnz = (double)Ly.nnz;
            const double act_bytes = 4.0 * Bc * (double)(nin + nout + (has_dprev ? nin : 0));
            prof_start(h, K_BWD, l, (is_fused ? 20.0 : 12.0) * nnz / nchunks + act_bytes,
                       (has_dprev ? 4.0 : 2.0) * nnz * Bc);
            SMLP_TRY(dispatch_bwd(h, A, Ly, has_dprev));
            prof_stop(h);
        }
    }
    return SMLP_OK;
}

int run_step(smlp_handle* h, const smlp_sgd* sgd) {
    const int threads = 256;
    const int64_t n = h->param_count;
    const int grid = (int)std::min<int64_t>((n + threads - 1) / threads, (int64_t)h->num_sms * 16);
    prof_start(h, K_SGD, 0, 20.0 * (double)n, 0.0);
    sgd_update_kernel<<<grid, threads, 0, h->stream>>>(h->param, h->mom, h->grad, n, h->bias_base, sgd->lr,
                                                       sgd->momentum, sgd->weight_decay, sgd->grad_scale);
    SMLP_CK_LAUNCH(h, "sgd_update_kernel");
    prof_stop(h);
    for (auto& Ly : h->layers) SMLP_TRY(refresh_mirror_values(h, Ly));
    return SMLP_OK;
}

}  // namespace smlp
