// step.cu — the per-minibatch hot path on sm_100a CUDA cores.
//
//   stage_input    a1  x[B x n_1] (optionally row-gathered by x_idx) -> act[1] chunked transposed
//   fwd_rows_kernel a2/a3  z_l = a_{l-1} W^(l) + b_l over the output-major mirror: one warp per
//                  <= SEG_NNZ-entry segment of an output row; G = CB/4 lanes hold one float4 of a
//                  gathered activation row, the P = 32/G groups take interleaved entries of the same
//                  row; the segment's (src, w) window is prefetched one segment ahead and staged in
//                  shared memory, 8 gather slots per lane are in flight before the first FMA (padding
//                  slots gather a zero row).  Epilogue: bias, All-ReLU (Eq. 3),
//                  inverted dropout (Philox), sign / keep bit masks.
//   fwd_finish     rows split into several segments: fixed-order sum of the partials + epilogue
//   softmax_ce     a3  p = softmax(z_L), loss, delta_L = (p - onehot)/B, output-bias gradient
//   bwd_rows_kernel a4/a5  one warp per segment of an input row i of the canonical CSR: per
//                  gathered delta_l[j] it accumulates delta_{l-1}[i] += w_ij delta_l[j] (SpMM against
//                  W^T) and the lane's partial of <a_{l-1}[i], delta_l[j]> (SDDMM), reduced per entry
//                  in a fixed order through shared memory; the gradient accumulates over chunks in the
//                  grad view; the Eq. 1 pass (sgd_update4) follows in the same API call
//   bits kernels   W^(2) when every input is 0 or 1: bit-packed input, exact sums of w / of delta
//   narrow kernels output layers with n_L <= 32: streamed canonical rows instead of gathers
//   bwd_finish     multi-segment rows: fixed-order sum of the delta partials + epilogue
//   sgd_update     a6 on the grad view (1 GPU: right after the backward; K > 1: after the allreduce),
//                  per layer slice, with each layer's mirror refresh on a side stream
//
// Batch chunks: with CB < B the batch is processed in ceil(B/CB) chunk launches so the gathered
// activation slab (n x CB fp32) stays L2-resident; gradients accumulate over chunks in order.
// No float atomics anywhere: every reduction has a fixed order, so results are deterministic.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>

#include "smlp_internal.cuh"

namespace smlp {
namespace {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ float4 ldg4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
__device__ __forceinline__ float4 f4zero() { return make_float4(0.f, 0.f, 0.f, 0.f); }
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

// L2 eviction policies (sm_80+ createpolicy / .L2::cache_hint): data streamed once per pass
// (indices, values, momenta, gradients) is marked evict_first so it does not push the gathered
// activation / delta slab of the chunk out of the L2; the gathers keep the normal policy.
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// read-only for the whole kernel
__device__ __forceinline__ float4 ldro_f4(const float* p, uint64_t pol) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p), "l"(pol));
    return v;
}
// read-write by the same thread within the kernel (coherent path)
__device__ __forceinline__ float ldrw_f32(const float* p, uint64_t pol) {
    float v;
    asm volatile("ld.global.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol) : "memory");
    return v;
}
__device__ __forceinline__ void st_f32(float* p, float v, uint64_t pol) {
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.f32 [%0], %1, %2;" :: "l"(p), "f"(v), "l"(pol) : "memory");
}

// L2-hinted variants used by the row kernels (hint = createpolicy register; "evict_normal" when the
// knob is off, so the instruction count is the same either way)
__device__ __forceinline__ float4 ldg4_hint(const float* p, uint64_t pol) {
    float4 v;
    asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ float ld_hint(const float* p, uint64_t pol) {
    float v;
    asm volatile("ld.global.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol) : "memory");
    return v;
}
__device__ __forceinline__ int ld_hint_i(const int32_t* p, uint64_t pol) {
    int v;
    asm volatile("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ void st_hint(float* p, float v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ float4 ld4_hint(const float* p, uint64_t pol) {   // coherent (read-write data)
    float4 v;
    asm volatile("ld.global.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p), "l"(pol) : "memory");
    return v;
}
__device__ __forceinline__ void st4_hint(float* p, float4 v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;"
                 ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol) : "memory");
}
__device__ __forceinline__ int4 ldi4_hint(const int32_t* p, uint64_t pol) {
    int4 v;
    asm volatile("ld.global.nc.L2::cache_hint.v4.s32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ uint64_t gather_policy(int hint) { return hint ? policy_evict_last() : policy_evict_normal(); }
__device__ __forceinline__ uint64_t stream_policy(int hint) { return hint ? policy_evict_first() : policy_evict_normal(); }

// Virtual grid of a kernel body ("persistent step"): every kernel of the step is a
// __device__ body run by 256-thread blocks with explicit block coordinates, called once by its
// own __global__ wrapper (vg = blockIdx / gridDim) or, for small models, by the persistent step
// kernel for each of the phase's virtual blocks in turn; shared memory comes from the caller.
struct VGrid {
    int bx, by, gx;
};
__device__ __forceinline__ VGrid hw_grid() { return VGrid{(int)blockIdx.x, (int)blockIdx.y, (int)gridDim.x}; }

// ------------------------------------------------------------------------------------------
// a1: input staging (transpose + optional row gather), zero padding of columns b >= B
// ------------------------------------------------------------------------------------------
// 32 batch rows x 128 features per block of 256 threads (8 warps x 4 sub-rows = 32 batch rows):
// float4 loads along the features (scalar when n_1 or x is not 16-B aligned), a shared-memory
// transpose (feature 4t + k stored at column 32k + t: conflict-free both ways), then per feature
// one coalesced row of the chunk layout and one 32-bit word of the bit-packed input
struct StageArgs {
    const float* x;
    const int32_t* x_idx;
    int B, nchunks, CB;
    int64_t n1;
    float* act1;
    uint32_t* xbits;
    int32_t* nonbinary;
    int vec;
};
struct StageSmem {
    float tile[32][129];
};
__device__ __forceinline__ void stage_input_body(const StageArgs& S, const VGrid vg, StageSmem& sm) {
    auto& tile = sm.tile;
    const int64_t f0 = (int64_t)vg.bx * 128;
    const int b0 = vg.by * 32;
    const int tx = threadIdx.x & 31;
#pragma unroll
    for (int sub = 0; sub < 4; ++sub) {
        const int ty = sub * 8 + (threadIdx.x >> 5);
        const int b = b0 + ty;
        const int64_t f = f0 + 4 * tx;
        float v[4] = {0.f, 0.f, 0.f, 0.f};
        if (b < S.B) {
            const int64_t row = S.x_idx ? (int64_t)__ldg(S.x_idx + b) : (int64_t)b;
            const float* p = S.x + row * S.n1 + f;
            if (S.vec && f + 3 < S.n1) {
                const float4 t = ldg4(p);
                v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (f + k < S.n1) v[k] = __ldg(p + k);
            }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) tile[ty][32 * k + tx] = v[k];
    }
    __syncthreads();
    const int b = b0 + tx;
#pragma unroll
    for (int sub = 0; sub < 4; ++sub) {
        const int ty = sub * 8 + (threadIdx.x >> 5);
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int fl = ty + 32 * r;                       // warp-uniform local feature
            const int64_t f = f0 + fl;
            const float v = tile[tx][32 * (fl & 3) + (fl >> 2)];
            if (f < S.n1 && b < S.nchunks * S.CB) {
                const int c = b / S.CB, lb = b % S.CB;
                S.act1[((int64_t)c * S.n1 + f) * S.CB + lb] = v;
            }
            if (S.xbits) {
                // the warp holds feature f over batch b0..b0+31: one 32-bit word of the bit-packed
                // input (bit b%32 = x[b][f] != 0) for the exact binary-input path of layer 2
                const unsigned word = __ballot_sync(FULL, v != 0.f);
                const bool nb = __any_sync(FULL, v != 0.f && v != 1.f);
                if (tx == 0 && f < S.n1) {
                    S.xbits[f * XBITS_WORDS + vg.by] = word;
                    if (nb) atomicOr(S.nonbinary, 1);
                }
            }
        }
    }
}
__global__ void __launch_bounds__(256) stage_input_kernel(StageArgs S) {
    SMLP_PDL_ENTRY();
    __shared__ StageSmem sm;
    stage_input_body(S, hw_grid(), sm);
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
    const int32_t* skip_if_binary;   // layer 2 with the binary-input path: return if *flag == 0
    int zero_row;                    // row index (relative to a_prev) of the zero row after the last chunk
    int l2hint;                      // L2 policies: gathers evict_last, streamed operands evict_first
    const int32_t* mrow_ptr;         // mirror row pointers (short-row streaming kernel)
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
    // dropout (R13): one Philox block per (neuron j, 4 batch rows): word c for row b0 + 4q + c
    const uint4 dr = A.dropout_on ? rng_stream(A.seed, P_DROPOUT, A.rank, A.layer, step_lo,
                                               ((uint64_t)j << 32) | (uint64_t)((A.b0 + q * 4) >> 2))
                                  : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const float zc = comp(z, c);
        const bool pos = zc > 0.f;
        zb[c] = group_bits<G>(__ballot_sync(FULL, own && pos), g);
        float a = pos ? zc : A.neg_slope * zc;
        bool keep = true;
        if (A.dropout_on) {
            keep = word(dr, c) >= A.drop_thr;
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



template <int CB>
__device__ __forceinline__ void fwd_finish_body(const FwdArgs& A, const VGrid vg) {
    constexpr int G = CB / 4, P = 32 / G;
    if (A.skip_if_binary && *A.skip_if_binary == 0) return;
    const int lane = threadIdx.x & 31, g = lane / G, q = lane % G;
    const int warp = (vg.bx * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (vg.gx * blockDim.x) >> 5;
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
template <int CB>
__global__ void __launch_bounds__(256) fwd_finish_kernel(FwdArgs A) {
    SMLP_PDL_ENTRY();
    fwd_finish_body<CB>(A, hw_grid());
}

// ------------------------------------------------------------------------------------------
// "row" kernels (default): one WARP per segment.  The P = 32/G groups of a warp take interleaved
// entries of the SAME row (entry e of a batch sits in slot u = e / P of group g = e % P), so no
// group idles while another finishes a longer row, and a whole batch of EB = U*P entries (64 for
// CB <= 32: a whole Poisson(40) row of C5) has its gathers in flight at once.  Each warp owns a
// contiguous range of segments, whose entry ranges are then contiguous too; the segment
// descriptor is loaded two segments ahead, the (index, weight) pairs and the row operand one
// segment ahead, so a row costs ~one gather round trip.  FMAs are packed (fma.rn.f32x2, bit-for-bit
// two fmaf).  Partial sums over the groups are combined by a fixed xor butterfly (every lane ends
// with the same bits), so results stay deterministic.
// ------------------------------------------------------------------------------------------
template <int CB, bool FWD = false>
struct RowCfg {
    static constexpr int G = CB / 4;                       // lanes per entry row (one float4 each)
    static constexpr int P = 32 / G;                       // entries per gather instruction
    // gather slots per batch: 8 x 16 B in flight per lane (more slots cost occupancy and measured
    // slower at every CB: profiles/spmm_bench_r01.txt, r01ae)
    static constexpr int UMAX = 8;
    static constexpr int U = (32 / P) < UMAX ? (32 / P) : UMAX;
    static constexpr int MINB = U > 12 ? 2 : (U > 8 ? 3 : 4);   // resident 256-thread blocks per SM
    static constexpr int EB = U * P;                       // entries per batch
    static constexpr int NW = SEG_NNZ / 32;                // window registers per lane (a segment = one window)
    static constexpr int NB = (SEG_NNZ + EB - 1) / EB;     // batches per window
    static constexpr int WIN = (NB * EB + 31) / 32 * 32;   // window slots in shared memory (>= SEG_NNZ)
    static constexpr int QS = U < 4 ? U : 4;               // slots per "quad" (issue granularity)
    static constexpr int NQ = U / QS;                      // quads per batch
    static constexpr int NR = P >= 4 ? 1 : 4 / P;          // epilogue components per lane
    static constexpr int S = G >= 8 ? G + 4 : G;           // smem stride of an entry's G partials
};
static_assert(SEG_NNZ % 32 == 0, "a segment is a whole number of 32-entry window registers");

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    float2 r;
    asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
        "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(r.x), "=f"(r.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return r;
}
// acc += w x (4 fmaf as 2 FFMA2)
__device__ __forceinline__ void fma4p(float4& acc, float w, const float4& x) {
    const float2 lo = ffma2(make_float2(w, w), make_float2(x.x, x.y), make_float2(acc.x, acc.y));
    const float2 hi = ffma2(make_float2(w, w), make_float2(x.z, x.w), make_float2(acc.z, acc.w));
    acc = make_float4(lo.x, lo.y, hi.x, hi.y);
}
// <a, x> over a lane's 4 columns in a fixed order: (a.x x.x + a.z x.z) + (a.y x.y + a.w x.w)
__device__ __forceinline__ float dot4p(const float4& a, const float4& x) {
    const float2 m = ffma2(make_float2(a.z, a.w), make_float2(x.z, x.w),
                           make_float2(a.x * x.x, a.y * x.y));
    return m.x + m.y;
}
__device__ __forceinline__ float4 f4add(const float4& a, const float4& b) {
    return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
__device__ __forceinline__ float4 shfl_xor4(const float4& v, int m) {
    return make_float4(__shfl_xor_sync(FULL, v.x, m), __shfl_xor_sync(FULL, v.y, m),
                       __shfl_xor_sync(FULL, v.z, m), __shfl_xor_sync(FULL, v.w, m));
}
// sum over the P groups of a warp (lanes q, q+G, q+2G, ...): fixed butterfly, identical in all lanes
template <int G>
__device__ __forceinline__ float4 group_allreduce(float4 v) {
#pragma unroll
    for (int m = G; m < 32; m <<= 1) v = f4add(v, shfl_xor4(v, m));
    return v;
}

// Sum of a float4 over the P groups of a warp, scattered: lane (g, q) ends with the components
// c = r P + g (r < NR) it finishes in the epilogue -- 3 shuffles for P = 4 instead of 8 for an
// all-reduce.  Fixed pairing, so the result is deterministic.
template <int CB>
__device__ __forceinline__ void group_reduce_scatter(float4 v, int g, float (&out)[RowCfg<CB>::NR]) {
    using C = RowCfg<CB>;
    constexpr int G = C::G, P = C::P;
    if constexpr (P == 1) {
        out[0] = v.x; out[1] = v.y; out[2] = v.z; out[3] = v.w;
    } else if constexpr (P == 2) {          // g = 0 keeps (x, z), g = 1 keeps (y, w)
        const bool hi = g & 1;
        const float k0 = hi ? v.y : v.x, k1 = hi ? v.w : v.z, s0 = hi ? v.x : v.y, s1 = hi ? v.z : v.w;
        out[0] = k0 + __shfl_xor_sync(FULL, s0, G);
        out[1] = k1 + __shfl_xor_sync(FULL, s1, G);
    } else {
#pragma unroll
        for (int m = 4 * G; m < 32; m <<= 1) v = f4add(v, shfl_xor4(v, m));   // groups beyond 4
        const bool b1 = (g & 2) != 0, b0 = (g & 1) != 0;
        const float ka = b1 ? v.z : v.x, kb = b1 ? v.w : v.y, sa = b1 ? v.x : v.z, sb = b1 ? v.y : v.w;
        const float pa = ka + __shfl_xor_sync(FULL, sa, 2 * G);   // component (g & 2) + 0
        const float pb = kb + __shfl_xor_sync(FULL, sb, 2 * G);   // component (g & 2) + 1
        const float keep = b0 ? pb : pa, send = b0 ? pa : pb;
        out[0] = keep + __shfl_xor_sync(FULL, send, G);           // component g & 3
    }
}

// cp.async (LDGSTS): global -> shared without a register destination, zero-filled when !valid
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src, bool valid, uint64_t pol) {
    asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 4, %2, %3;" ::"r"(dst), "l"(src),
                 "r"(valid ? 4 : 0), "l"(pol) : "memory");
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid, uint64_t pol) {
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2, %3;" ::"r"(dst), "l"(src),
                 "r"(valid ? 16 : 0), "l"(pol) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// Segment pipeline of the row kernels: the (index, weight) window of segment [beg, end)
// (<= SEG_NNZ entries) goes to the warp's shared-memory buffer as int2 (row, weight bits) by
// cp.async one segment ahead, so the prefetch holds no registers.  Entries past the end are
// zero-filled and then pointed at the zero row after the last chunk (weight 0), so every gather
// slot of a quad is unconditional.
__device__ __forceinline__ void window_async(int2* win, const int32_t* __restrict__ idx, const float* __restrict__ wv,
                                             int beg, int end, int lane, uint64_t pol) {
#pragma unroll
    for (int r = 0; r < SEG_NNZ / 32; ++r) {
        const int e = lane + 32 * r, k = beg + e;
        const bool ok = k < end;
        cp_async4(smem_u32(&win[e].x), idx + (ok ? k : beg), ok, pol);
        cp_async4(smem_u32(&win[e].y), wv + (ok ? k : beg), ok, pol);
    }
}
__device__ __forceinline__ void window_pad(int2* win, int n, int lane, int zero_row) {
#pragma unroll
    for (int r = 0; r < SEG_NNZ / 32; ++r) {
        const int e = lane + 32 * r;
        if (e >= n) win[e].x = zero_row;
    }
}

// forward epilogue of one complete row j (acc = the row's sum, identical in every lane): lane
// (g, q) finishes components c = r P + g of its float4 (columns 4q + c), so all 32 lanes share
// the bias / All-ReLU / dropout / mask work and the store is one coalesced row.
template <int CB>
__device__ __forceinline__ void fwd_rows_epilogue_c(const FwdArgs& A, int64_t j, const float (&zr)[RowCfg<CB, true>::NR],
                                                    float bj, int lane, uint32_t step_lo) {
    using C = RowCfg<CB, true>;
    constexpr int G = C::G, P = C::P, NR = C::NR;
    const int g = lane / G, q = lane % G;
    uint32_t bal_p[NR], bal_k[NR];
    // dropout (R13): one Philox block per (neuron j, 4 batch rows): word c for row b0 + 4q + c
    const uint4 dr = (A.hidden && A.dropout_on)
                         ? rng_stream(A.seed, P_DROPOUT, A.rank, A.layer, step_lo,
                                      ((uint64_t)j << 32) | (uint64_t)((A.b0 + q * 4) >> 2))
                         : make_uint4(0, 0, 0, 0);
    float out[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) {
        const int c = r * P + g;
        const bool valid = c < 4;
        const float z = zr[r] + bj;
        if (!A.hidden) {
            out[r] = z;
            continue;
        }
        const bool pos = z > 0.f;
        float a = pos ? z : A.neg_slope * z;
        bool keep = true;
        if (A.dropout_on && valid) {
            keep = word(dr, c & 3) >= A.drop_thr;
            a = keep ? a * A.keep_scale : 0.f;
        }
        out[r] = a;
        bal_p[r] = __ballot_sync(FULL, valid && pos);
        bal_k[r] = __ballot_sync(FULL, valid && keep);
    }
    if constexpr (P == 1) {   // the lane holds its 4 columns: one 16-B store
        st4(A.a_out + j * CB + q * 4, make_float4(out[0], out[1], out[2], out[3]));
    } else {
#pragma unroll
        for (int r = 0; r < NR; ++r) {
            const int c = r * P + g;
            if (c < 4) A.a_out[j * CB + q * 4 + c] = out[r];
        }
    }
    if (A.hidden && lane == 0) {
        uint32_t zb[4], kb[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {   // word c, bit q = column 4q + c, held by group c % P of ballot c / P
            zb[c] = group_bits<G>(bal_p[(c / P) % NR], c % P);
            kb[c] = group_bits<G>(bal_k[(c / P) % NR], c % P);
        }
        A.zmask[j] = make_uint4(zb[0], zb[1], zb[2], zb[3]);
        if (A.dropout_on) A.kmask[j] = make_uint4(kb[0], kb[1], kb[2], kb[3]);
    }
}

// the same with the row's complete float4 in every lane
template <int CB>
__device__ __forceinline__ void fwd_rows_epilogue(const FwdArgs& A, int64_t j, const float4& acc, float bj, int lane,
                                                  uint32_t step_lo) {
    using C = RowCfg<CB, true>;
    float zr[C::NR];
#pragma unroll
    for (int r = 0; r < C::NR; ++r) zr[r] = comp(acc, (r * C::P + lane / C::G) & 3);
    fwd_rows_epilogue_c<CB>(A, j, zr, bj, lane, step_lo);
}

// NS gather slots of a batch, all issued before the first FMA (entry u P + g of the window in slot u)
template <int CB, int NS>
__device__ __forceinline__ void fwd_slots(const float* __restrict__ a_prev, const int2* win, int g, int q,
                                          float4& acc, uint64_t pg) {
    constexpr int P = RowCfg<CB, true>::P;
    float4 x[NS];
    float wv[NS];
#pragma unroll
    for (int u = 0; u < NS; ++u) {
        const int2 e = win[u * P + g];
        wv[u] = __int_as_float(e.y);
        x[u] = ldg4_hint(a_prev + (int64_t)e.x * CB + q * 4, pg);
    }
#pragma unroll
    for (int u = 0; u < NS; ++u) fma4p(acc, wv[u], x[u]);
}

// one batch of nb <= EB entries: the smallest number of quads covering it (warp-uniform switch,
// one fully unrolled body per length class; the padding slots gather the zero row)
template <int CB>
__device__ __forceinline__ void fwd_batch(const float* __restrict__ a_prev, const int2* win, int nb, int g, int q,
                                          float4& acc, uint64_t pg) {
    using C = RowCfg<CB, true>;
    if constexpr (C::NQ == 1) {
        fwd_slots<CB, C::QS>(a_prev, win, g, q, acc, pg);
    } else {
        if (nb > C::QS * C::P) fwd_slots<CB, C::U>(a_prev, win, g, q, acc, pg);
        else fwd_slots<CB, C::QS>(a_prev, win, g, q, acc, pg);
    }
}

// register-prefetched window (the forward keeps its LSU for the gathers: no LDGSTS)
template <int NW>
__device__ __forceinline__ void load_window(const int32_t* __restrict__ idx, const float* __restrict__ wv, int beg,
                                            int end, int lane, int (&ix)[NW], float (&w)[NW]) {
#pragma unroll
    for (int r = 0; r < NW; ++r) {
        const int k = beg + lane + 32 * r;
        ix[r] = k < end ? __ldg(idx + k) : 0;
        w[r] = k < end ? __ldg(wv + k) : 0.f;
    }
}
template <int NW>
__device__ __forceinline__ void stage_window(int2* win, const int (&ix)[NW], const float (&w)[NW], int n, int lane,
                                             int zero_row) {
#pragma unroll
    for (int r = 0; r < NW; ++r) {
        const int e = lane + 32 * r;
        win[e] = e < n ? make_int2(ix[r], __float_as_int(w[r])) : make_int2(zero_row, 0);
    }
}

template <int CB>
struct FwdRowsSmem {
    __align__(16) int2 win_all[WARPS_PER_BLOCK][RowCfg<CB, true>::WIN];
};
template <int CB>
__device__ __forceinline__ void fwd_rows_body(const FwdArgs& A, const VGrid vg, FwdRowsSmem<CB>& sm) {
    using C = RowCfg<CB, true>;
    constexpr int G = C::G, EB = C::EB, NW = C::NW, NB = C::NB;
    auto& win_all = sm.win_all;
    if (A.skip_if_binary && *A.skip_if_binary == 0) return;
    const int lane = threadIdx.x & 31, g = lane / G, q = lane % G;
    int2* win = win_all[threadIdx.x >> 5];
    for (int e = SEG_NNZ + lane; e < C::WIN; e += 32) win[e] = make_int2(A.zero_row, 0);   // never-used tail
    const uint64_t pg = gather_policy(A.l2hint);
    const int64_t warp = ((int64_t)vg.bx * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)vg.gx * blockDim.x) >> 5;
    const int64_t nseg = A.meta->n_fseg;
    const int64_t s_lo = warp * nseg / nwarps, s_hi = (warp + 1) * nseg / nwarps;
    if (s_lo >= s_hi) return;
    const uint32_t step_lo = A.step_ptr ? (uint32_t)(*A.step_ptr) : A.step_lo;
    const int4 none = make_int4(0, 0, 0, -2);
    int4 cur = A.seg[s_lo];
    int4 nxt = s_lo + 1 < s_hi ? A.seg[s_lo + 1] : none;
    int ix[NW];
    float w[NW];
    load_window<NW>(A.msrc, A.mval, cur.y, cur.z, lane, ix, w);
    for (int64_t s = s_lo; s < s_hi; ++s) {
        const int4 nn = s + 2 < s_hi ? A.seg[s + 2] : none;      // descriptor two ahead
        int ix_n[NW];
        float w_n[NW];
        load_window<NW>(A.msrc, A.mval, nxt.y, nxt.z, lane, ix_n, w_n);   // indices one ahead
        const float bj = cur.w < 0 ? __ldg(A.bias + cur.x) : 0.f;         // consumed after the gathers
        const int n = cur.z - cur.y;
        SMLP_BOUND(0 <= cur.y && cur.y <= cur.z && cur.z <= A.meta->nnz && n <= SEG_NNZ, "fwd segment");
#pragma unroll
        for (int r = 0; r < NW; ++r)
            SMLP_BOUND(lane + 32 * r >= n || (unsigned)ix[r] < (unsigned)A.zero_row, "fwd gathered row");
        __syncwarp();
        stage_window<NW>(win, ix, w, n, lane, A.zero_row);
        __syncwarp();
        float4 acc = f4zero();
#pragma unroll
        for (int b = 0; b < NB; ++b)
            if (b * EB < n) fwd_batch<CB>(A.a_prev, win + b * EB, n - b * EB, g, q, acc, pg);
        if (cur.w < 0) {
            float zr[C::NR];
            group_reduce_scatter<CB>(acc, g, zr);
            fwd_rows_epilogue_c<CB>(A, cur.x, zr, bj, lane, step_lo);
        } else {
            acc = group_allreduce<G>(acc);
            if (g == 0) st4(A.ws + (int64_t)cur.w * CB + q * 4, acc);
        }
        cur = nxt;
        nxt = nn;
#pragma unroll
        for (int r = 0; r < NW; ++r) {
            ix[r] = ix_n[r];
            w[r] = w_n[r];
        }
    }
}
template <int CB>
__global__ void __launch_bounds__(256, RowCfg<CB, true>::MINB) fwd_rows_kernel(FwdArgs A) {
    SMLP_PDL_ENTRY();
    __shared__ FwdRowsSmem<CB> sm;
    fwd_rows_body<CB>(A, hw_grid(), sm);
}

// Short-row forward (128-column chunks, rows averaging < 16 entries: Table 4's eps <= 5 layers).
// The row kernel above spends one window / descriptor / batch round per row and has ~2 gathers
// in flight per warp there.  This one streams a unit of 32 consecutive mirror rows as one entry
// range: lane t loads entry t of each 32-entry block (coalesced), and the warp gathers 8 entries'
// rows at a time across row boundaries (the lane's float4 = its 4 columns), then consumes them in
// order, finishing each row (fwd_rows_epilogue) as its last entry is added -- the same sequential
// sum per row as the row kernel, so the result is identical.
constexpr int SHORT_ROWS = 32;
__global__ void __launch_bounds__(256, 4) fwd_short_rows_kernel(FwdArgs A) {
    SMLP_PDL_ENTRY();
    constexpr int CB = 128, GU = 4;                 // gathers in flight per warp (4 x 16 B, 64 regs)
    __shared__ int2 rec_all[WARPS_PER_BLOCK][32 + GU];
    if (A.skip_if_binary && *A.skip_if_binary == 0) return;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    int2* rec = rec_all[wib];
    if (lane < GU) rec[32 + lane] = make_int2(A.zero_row, 0);          // never-consumed tail
    const uint64_t pg = gather_policy(A.l2hint), ps = stream_policy(A.l2hint);
    const uint32_t step_lo = A.step_ptr ? (uint32_t)(*A.step_ptr) : A.step_lo;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t nunits = (A.n_out + SHORT_ROWS - 1) / SHORT_ROWS;
    for (int64_t u0 = warp; u0 < nunits; u0 += nwarps) {
        const int64_t j0 = u0 * SHORT_ROWS;
        const int nrows = (int)(A.n_out - j0 < SHORT_ROWS ? A.n_out - j0 : SHORT_ROWS);
        const int rp_l = __ldg(A.mrow_ptr + j0 + min(lane, nrows));      // lane t: start of local row t
        const float b_l = lane < nrows ? __ldg(A.bias + j0 + lane) : 0.f;
        const int E0 = __shfl_sync(FULL, rp_l, 0), E1 = __ldg(A.mrow_ptr + j0 + nrows);
        int row = 0;
        int row_end = nrows > 1 ? __shfl_sync(FULL, rp_l, 1) : E1;
        float4 acc = f4zero();
        auto finish_rows_at = [&](int e) {          // finish every row ending at entry e (empty rows too)
            while (row < nrows && e == row_end) {
                fwd_rows_epilogue<CB>(A, j0 + row, acc, __shfl_sync(FULL, b_l, row), lane, step_lo);
                acc = f4zero();
                ++row;
                row_end = row + 1 < nrows ? __shfl_sync(FULL, rp_l, min(row + 1, 31)) : E1;
            }
        };
        for (int blk = E0; blk < E1; blk += 32) {
            const int n = min(32, E1 - blk);
            __syncwarp();
            rec[lane] = lane < n ? make_int2(ld_hint_i(A.msrc + blk + lane, ps), __float_as_int(ld_hint(A.mval + blk + lane, ps)))
                                 : make_int2(A.zero_row, 0);
            SMLP_BOUND((unsigned)rec[lane].x <= (unsigned)A.zero_row, "fwd short gathered row");
            __syncwarp();
            for (int v0 = 0; v0 < n; v0 += GU) {
                float4 x[GU];
                float wv[GU];
#pragma unroll
                for (int k = 0; k < GU; ++k) {      // GU rows in flight, across row boundaries
                    const int2 e = rec[v0 + k];
                    wv[k] = __int_as_float(e.y);
                    x[k] = ldg4_hint(A.a_prev + (int64_t)e.x * CB + lane * 4, pg);
                }
                // consume in order, one row segment at a time (one epilogue call site): entries
                // k .. stop-1 of this group belong to the current row
                const int kmax = min(GU, n - v0);
                int k = 0;
                for (;;) {
                    finish_rows_at(blk + v0 + k);
                    if (k >= kmax) break;
                    const int stop = min(kmax, row_end - (blk + v0));
#pragma unroll
                    for (int kk = 0; kk < GU; ++kk)
                        if (kk >= k && kk < stop) fma4p(acc, wv[kk], x[kk]);
                    k = stop;
                }
            }
        }
        finish_rows_at(E1);
    }
}

// ------------------------------------------------------------------------------------------
// softmax cross-entropy (single block, fixed-order reductions)
// ------------------------------------------------------------------------------------------
struct SoftmaxArgs {
    const float* logits;      // act[L] [nchunks_f][n_L][CBf]
    float* delta;             // delta[L] [nchunks][n_L][CB]
    const int32_t* labels;
    const int32_t* y_idx;
    float* loss;              // scalar or null
    int32_t* err;
    float* bias;              // b_L
    float* bias_mom;
    float* bias_grad;         // grad view slice (unfused)
    int64_t nL;
    int B, nchunks, CB, CBf;
    int fused;
    float lr, mu;
};

// One block of 256 threads standing in for the 512 virtual threads of the loss tree: thread t
// takes batch columns b = t, t + 512, ... (virtual thread t) and b = t + 256, t + 768, ...
// (virtual thread t + 256); red[t] = their two fp64 sums is the 512-tree's first level, the rest
// of the tree follows in the same fixed order.
struct SoftmaxSmem {
    double red[256];
};
__device__ __forceinline__ double softmax_ce_cols(const SoftmaxArgs& A, int v) {
    double lsum = 0.0;
    const int total = A.nchunks * A.CB;
    const float invB = 1.0f / (float)A.B;
    for (int b = v; b < total; b += 512) {
        const int c = b / A.CB, lb = b % A.CB;
        const float* zc = A.logits + (int64_t)(b / A.CBf) * A.nL * A.CBf + b % A.CBf;
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
        for (int64_t j = 0; j < A.nL; ++j) mx = fmaxf(mx, zc[j * A.CBf]);
        float s = 0.f;
        for (int64_t j = 0; j < A.nL; ++j) s += expf(zc[j * A.CBf] - mx);
        const float lse = logf(s);
        lsum += (double)(lse - (zc[(int64_t)y * A.CBf] - mx));
        const float inv = 1.0f / s;
        for (int64_t j = 0; j < A.nL; ++j) {
            const float p = expf(zc[j * A.CBf] - mx) * inv;
            dc[j * A.CB] = (p - (j == y ? 1.f : 0.f)) * invB;
        }
    }
    return lsum;
}
__device__ __forceinline__ void softmax_ce_body(const SoftmaxArgs& A, SoftmaxSmem& sm) {
    double* red = sm.red;
    const int tid = threadIdx.x;
    const double l0 = softmax_ce_cols(A, tid), l1 = softmax_ce_cols(A, tid + 256);
    red[tid] = l0 + l1;
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if (tid < s) red[tid] += red[tid + s];
        __syncthreads();
    }
    if (tid == 0 && A.loss) *A.loss = (float)(red[0] / (double)A.B);
    // output-layer bias gradient gb_L = sum_b delta_L[b, :]
    for (int64_t j = tid; j < A.nL; j += 256) {
        float g = 0.f;
        for (int c = 0; c < A.nchunks; ++c) {
            const float* dc = A.delta + ((int64_t)c * A.nL + j) * A.CB;
            for (int lb = 0; lb < A.CB; ++lb) g += dc[lb];
        }
        A.bias_grad[j] = g;
    }
}
__global__ void __launch_bounds__(256) softmax_ce_kernel(SoftmaxArgs A) {
    SMLP_PDL_ENTRY();
    __shared__ SoftmaxSmem sm;
    softmax_ce_body(A, sm);
}

__global__ void softmax_probs_kernel(const float* __restrict__ logits, float* __restrict__ probs, int64_t nL, int B,
                                     int CB) {
    SMLP_PDL_ENTRY();
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
    const float* a_prev;      // a_{l-1}, forward layout: base of forward chunk c CB / CBF ([n_in][CBF] each)
    const float* d_out;       // chunk base [n_out][CB]  (delta_l)
    float* d_prev;            // chunk base [n_in][CB]   (delta_{l-1}) or null for l = 2
    const uint4* zmask_prev;  // forward layout: base of forward chunk c CB / CBF ([n_in] each)
    const uint4* kmask_prev;
    int64_t n_prev;           // n_{l-1}
    const int4* seg;
    const int4* multi;
    const LayerMeta* meta;
    const int32_t* col;
    float* val;
    float* mom;
    float* grad;
    float* mval;              // mirror-ordered copy of w (refreshed by the fused update)
    const int32_t* minv;      // canonical index -> mirror position
    int mval_scatter;         // the fused update also scatters w into mval (no separate refresh)
    float* ws;
    float* bgs;               // [n_in] bias-grad accumulator over chunks
    float* bias_prev;
    float* bias_mom_prev;
    float* bias_grad_prev;
    float neg_slope_prev;
    float keep_scale_prev;
    int dropout_prev;
    int first, last;          // first / last chunk processed for this layer (grad accumulation)
    int no_gold;              // the last chunk writes its own gradient buffer (the Eq. 1 pass adds both)
    int fused;
    float lr, mu, wd;
    const int32_t* skip_if_binary;   // layer 2 with the binary-input path: return if *flag == 0
    int zero_row;                    // row index (relative to d_out) of the zero row after the last chunk
    int l2hint;                      // L2 policies: gathers evict_last, streamed operands evict_first
    const int32_t* row_ptr;          // canonical row pointers (short-row streaming kernel)
    const int32_t* rowid;            // canonical row of each entry (short-row streaming kernel)
    // implicit delta_l (l = L-1 under a dense-capped 2-output layer, RECOMP kernels): per-neuron records
    // (sign bits of the chunk's columns, w_j0, w_j1), delta_L of the chunk [2][CB], and the negative
    // slope of layer l's activation; zero_row then indexes the all-zero record
    const uint4* drec;
    const float* dL;
    float rc_slope;
};

// Forward-layout position of a backward chunk's local column lc (CB = R CBF, R in {1, 2, 4}; the
// chunk base passed is that of forward chunk c R): column lc lives in forward chunk c R + lc / CBF
// at column off = lc % CBF, so a_{l-1}[i] of it is a_prev[i CBF + aoff] and its mask bits are word
// off & 3, bit off >> 2 of zmask_prev[i + moff].  With CBF = CB: aoff = lc, moff = 0, the plain
// layout (compile-time).
template <int CB, int CBF>
struct FwdPos {
    int64_t aoff, moff;
    int off;
    __device__ __forceinline__ FwdPos(int lc, int64_t n) {
        if constexpr (CBF == CB) {
            aoff = lc; moff = 0; off = lc;
        } else {
            off = lc % CBF;
            moff = (int64_t)(lc / CBF) * n;
            aoff = moff * CBF + off;
        }
    }
};

// delta_{l-1} of input row i per group: f'(z) from the sign bits, dropout keep bits, store, and
// the bias gradient of layer l-1 (accumulated across chunks in order).
template <int CB, int CBF>
__device__ __forceinline__ void bwd_epilogue(const BwdArgs& A, int64_t i, float4 d, bool own, int lane) {
    constexpr int G = CB / 4;
    const int q = lane % G;
    float o[4] = {0.f, 0.f, 0.f, 0.f};
    if (own) {
        const FwdPos<CB, CBF> fp(4 * q, A.n_prev);
        const int qb = fp.off >> 2;
        const uint4 zb = A.zmask_prev[fp.moff + i];
        uint4 kb = make_uint4(FULL, FULL, FULL, FULL);
        if (A.dropout_prev) kb = A.kmask_prev[fp.moff + i];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const bool pos = (word(zb, c) >> qb) & 1u;
            const bool keep = (word(kb, c) >> qb) & 1u;
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
        if (!A.first) tot += A.bgs[i];
        if (!A.last) A.bgs[i] = tot;
        else A.bias_grad_prev[i] = tot;
    }
}


template <int CB, int CBF>
__device__ __forceinline__ void bwd_finish_body(const BwdArgs& A, const VGrid vg) {
    constexpr int G = CB / 4, P = 32 / G;
    if (A.skip_if_binary && *A.skip_if_binary == 0) return;
    const int lane = threadIdx.x & 31, g = lane / G, q = lane % G;
    const int warp = (vg.bx * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (vg.gx * blockDim.x) >> 5;
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
        bwd_epilogue<CB, CBF>(A, m.x, acc, active, lane);
    }
}
template <int CB, int CBF>
__global__ void __launch_bounds__(256) bwd_finish_kernel(BwdArgs A) {
    SMLP_PDL_ENTRY();
    bwd_finish_body<CB, CBF>(A, hw_grid());
}

// backward epilogue of one complete input row i (d = sum_j w_ij delta_l[j], identical in every
// lane): f'_{l-1} from the sign bits, dropout keep bits, store of delta_{l-1}[i], and the bias
// gradient of layer l-1 (a fixed 32-lane butterfly, then accumulated over chunks in order)
struct BwdSide {            // per-row operands of the backward epilogue (loaded before the gathers)
    uint4 zb, kb;           // sign / keep bits of layer l-1, row i
    float bgs;              // lane 0: bias-grad accumulator of neuron i
};
template <bool DROP>
__device__ __forceinline__ BwdSide bwd_side(const BwdArgs& A, int64_t i, int64_t moff, bool valid, int lane) {
    BwdSide t;
    t.zb = make_uint4(0, 0, 0, 0);
    t.kb = make_uint4(FULL, FULL, FULL, FULL);
    t.bgs = 0.f;
    if (!valid) return t;
    t.zb = A.zmask_prev[moff + i];
    if (DROP) t.kb = A.kmask_prev[moff + i];
    if (lane == 0 && !A.first) t.bgs = A.bgs[i];
    return t;
}

// backward epilogue of one complete input row i: f'_{l-1} from the sign bits, dropout keep bits,
// store of delta_{l-1}[i], and the bias gradient of layer l-1 (a fixed 32-lane butterfly, then
// accumulated over chunks in order).  d[r] = component r P + g of the row's sum.
template <int CB>
__device__ __forceinline__ void bwd_rows_epilogue(const BwdArgs& A, int64_t i, const float (&d)[RowCfg<CB>::NR],
                                                  const BwdSide& sd, int qb, int lane) {
    using C = RowCfg<CB>;
    constexpr int G = C::G, P = C::P, NR = C::NR;
    const int g = lane / G, q = lane % G;
    const uint4 zb = sd.zb, kb = sd.kb;
    float s = 0.f;
    float out[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) {
        const int c = r * P + g;
        out[r] = 0.f;
        if (c < 4) {
            const bool pos = (word(zb, c) >> qb) & 1u;
            const bool keep = (word(kb, c) >> qb) & 1u;
            const float v = d[r] * (pos ? 1.f : A.neg_slope_prev);
            const float o = A.dropout_prev ? (keep ? v * A.keep_scale_prev : 0.f) : v;
            out[r] = o;
            s += o;
        }
    }
    if constexpr (P == 1) {   // the lane holds its 4 columns: one 16-B store
        st4(A.d_prev + i * CB + q * 4, make_float4(out[0], out[1], out[2], out[3]));
    } else {
#pragma unroll
        for (int r = 0; r < NR; ++r) {
            const int c = r * P + g;
            if (c < 4) A.d_prev[i * CB + q * 4 + c] = out[r];
        }
    }
#pragma unroll
    for (int m = 1; m < 32; m <<= 1) s += __shfl_xor_sync(FULL, s, m);
    if (lane == 0) {
        float tot = s;
        if (!A.first) tot += sd.bgs;
        if (!A.last) A.bgs[i] = tot;
        else A.bias_grad_prev[i] = tot;
    }
}

// operands of the implicit delta_l (RECOMP): delta_L of the lane's 4 columns, the slope, and where
// the lane's sign bits sit in a record
struct Recomp {
    float4 d0, d1;
    float slope;
    int sh;          // bit position of the lane's first column in its sign word
    bool hi;         // the lane's columns are 32..63 (second sign word)
};
// delta_l[j] of the lane's 4 columns from neuron j's record: f'(z) (w_j0 delta_L[0] + w_j1 delta_L[1]),
// the expression (and rounding) of bwd_narrow_rows_body; x 1 is skipped (exact)
__device__ __forceinline__ float4 recomp_delta(const uint4& rc, const Recomp& R) {
    const float w0 = __uint_as_float(rc.z), w1 = __uint_as_float(rc.w);
    // the lane's 4 sign bits rotated onto bits 1..4: one register-to-predicate move sets all four
    const uint32_t sw = R.hi ? rc.y : rc.x;
    const uint32_t nib = __funnelshift_r(sw, sw, (R.sh + 31) & 31);
    // fmaf(w1, d1, fmaf(w0, d0, 0)) per column, two columns per FFMA2 (bit for bit two fmaf)
    const float2 z2 = make_float2(0.f, 0.f), w00 = make_float2(w0, w0), w11 = make_float2(w1, w1);
    const float2 lo = ffma2(w11, make_float2(R.d1.x, R.d1.y), ffma2(w00, make_float2(R.d0.x, R.d0.y), z2));
    const float2 hh = ffma2(w11, make_float2(R.d1.z, R.d1.w), ffma2(w00, make_float2(R.d0.z, R.d0.w), z2));
    float4 d = make_float4(lo.x, lo.y, hh.x, hh.y);
    if (!(nib & 2u)) d.x *= R.slope;
    if (!(nib & 4u)) d.y *= R.slope;
    if (!(nib & 8u)) d.z *= R.slope;
    if (!(nib & 16u)) d.w *= R.slope;
    return d;
}

template <int CB, int NS, bool HAS_DPREV, bool RECOMP>
__device__ __forceinline__ void bwd_slots(const float* __restrict__ d_out, const int2* win, float* red,
                                          const float4& ai, int g, int q, float4& dacc, uint64_t pg,
                                          const uint4* rec, const Recomp& R) {
    using C = RowCfg<CB>;
    constexpr int P = C::P, S = C::S;
    float4 dx[NS];
    float wv[NS];
#pragma unroll
    for (int u = 0; u < NS; ++u) {
        const int2 e = win[u * P + g];
        wv[u] = __int_as_float(e.y);
        if constexpr (RECOMP) dx[u] = recomp_delta(rec[u * P + g], R);   // the entry's record, staged by the row loop
        else dx[u] = ldg4_hint(d_out + (int64_t)e.x * CB + q * 4, pg);
    }
#pragma unroll
    for (int u = 0; u < NS; ++u) {
        if (HAS_DPREV) fma4p(dacc, wv[u], dx[u]);
#if !SMLP_EXP_NO_SDDMM
        red[(u * P + g) * S + q] = dot4p(ai, dx[u]);     // entry u P + g of this batch: lane-q partial
#endif
    }
}

template <int CB, bool HAS_DPREV, bool RECOMP>
__device__ __forceinline__ void bwd_batch(const float* __restrict__ d_out, const int2* win, float* red, int nb,
                                          const float4& ai, int g, int q, float4& dacc, uint64_t pg,
                                          const uint4* rec, const Recomp& R) {
    using C = RowCfg<CB>;
    if constexpr (RECOMP && C::NQ == 2) {
        // records come from shared memory: nothing in flight to keep, so a quad at a time (half the
        // registers of a full batch; same entries, same order)
        bwd_slots<CB, C::QS, HAS_DPREV, RECOMP>(d_out, win, red, ai, g, q, dacc, pg, rec, R);
        if (nb > C::QS * C::P)
            bwd_slots<CB, C::QS, HAS_DPREV, RECOMP>(d_out, win + C::QS * C::P, red + C::QS * C::P * C::S, ai, g, q, dacc,
                                                    pg, rec + C::QS * C::P, R);
    } else if constexpr (C::NQ == 1) {
        bwd_slots<CB, C::QS, HAS_DPREV, RECOMP>(d_out, win, red, ai, g, q, dacc, pg, rec, R);
    } else {
        if (nb > C::QS * C::P) bwd_slots<CB, C::U, HAS_DPREV, RECOMP>(d_out, win, red, ai, g, q, dacc, pg, rec, R);
        else bwd_slots<CB, C::QS, HAS_DPREV, RECOMP>(d_out, win, red, ai, g, q, dacc, pg, rec, R);
    }
}

// GOLD: add the gradient accumulated by earlier chunks; DROP: dropout on layer l-1
template <int CB>
struct BwdRowsSmem {
    static constexpr int RB = RowCfg<CB>::NB < 2 ? RowCfg<CB>::NB : 2;   // batches per reduction round
    __align__(16) int2 win_all[WARPS_PER_BLOCK][2][SEG_NNZ];
    __align__(16) float4 ai_all[WARPS_PER_BLOCK][2][RowCfg<CB>::G];
    __align__(16) float red_all[WARPS_PER_BLOCK][RB * RowCfg<CB>::EB * RowCfg<CB>::S];
};
// per-warp staging of a segment's records (RECOMP kernels only)
struct BwdRecSmem {
    __align__(16) uint4 rec_all[WARPS_PER_BLOCK][SEG_NNZ];
};
template <int CB, int CBF, bool HAS_DPREV, bool GOLD, bool DROP, bool RECOMP = false>
__device__ __forceinline__ void bwd_rows_body(const BwdArgs& A, const VGrid vg, BwdRowsSmem<CB>& sm,
                                              BwdRecSmem* rsm = nullptr) {
    using C = RowCfg<CB>;
    constexpr int G = C::G, EB = C::EB, NW = C::NW, NB = C::NB, S = C::S, NR = C::NR;
    constexpr int RB = BwdRowsSmem<CB>::RB;
    auto& win_all = sm.win_all;
    auto& ai_all = sm.ai_all;
    auto& red_all = sm.red_all;
    if (A.skip_if_binary && *A.skip_if_binary == 0) return;
    const int lane = threadIdx.x & 31, g = lane / G, q = lane % G;
    const int wib = threadIdx.x >> 5;
    int2 (*win)[SEG_NNZ] = win_all[wib];
    float4 (*ais)[G] = ai_all[wib];
    float* red = red_all[wib];
    const int64_t warp = ((int64_t)vg.bx * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)vg.gx * blockDim.x) >> 5;
    const int64_t nseg = A.meta->n_bseg;
    const int64_t s_lo = warp * nseg / nwarps, s_hi = (warp + 1) * nseg / nwarps;
    if (s_lo >= s_hi) return;
    const int4 none = make_int4(0, 0, 0, -2);
    const uint64_t pg = gather_policy(A.l2hint), ps = stream_policy(A.l2hint);
    const FwdPos<CB, CBF> fp(4 * q, A.n_prev);   // the lane's 4 columns in the forward layout
    Recomp R{};
    uint4* rec = nullptr;
    if constexpr (RECOMP) {
        R.d0 = ldg4(A.dL + q * 4);
        R.d1 = ldg4(A.dL + CB + q * 4);
        R.slope = A.rc_slope;
        R.sh = (4 * q) & 31;
        R.hi = 4 * q >= 32;
        rec = rsm->rec_all[wib];
    }
    // window + a_{l-1}[i] of a segment into buffer b (cp.async, one segment ahead: no registers held)
    auto prefetch = [&](const int4& sg, int b) {
        window_async(win[b], A.col, A.val, sg.y, sg.z, lane, ps);
        if (lane < G)
            cp_async16(smem_u32(&ais[b][lane]), A.a_prev + (int64_t)(sg.w != -2 ? sg.x : 0) * CBF + fp.aoff, sg.w != -2,
                       ps);
        cp_async_commit();
    };
    int4 cur = A.seg[s_lo];
    int4 nxt = s_lo + 1 < s_hi ? A.seg[s_lo + 1] : none;
    prefetch(cur, 0);
    int buf = 0;
    for (int64_t s = s_lo; s < s_hi; ++s) {
        const int4 nn = s + 2 < s_hi ? A.seg[s + 2] : none;
        prefetch(nxt, buf ^ 1);
        // operands consumed after the gathers: the lane's entries' earlier-chunk gradient, and the
        // row's epilogue side data
        const int n = cur.z - cur.y;
        float gold[NW];
#pragma unroll
        for (int r = 0; r < NW; ++r) {
            const int k = cur.y + lane + 32 * r;
            const bool ok = lane + 32 * r < n;
            gold[r] = GOLD && ok ? ld_hint(A.grad + k, ps) : 0.f;
        }
        const BwdSide sd = bwd_side<DROP>(A, cur.x, fp.moff, HAS_DPREV && cur.w < 0, lane);
        cp_async_wait1();
        __syncwarp();
        window_pad(win[buf], n, lane, A.zero_row);
        SMLP_BOUND(0 <= cur.y && cur.y <= cur.z && cur.z <= A.meta->nnz && n <= SEG_NNZ, "bwd segment");
#pragma unroll
        for (int r = 0; r < SEG_NNZ / 32; ++r)
            SMLP_BOUND((unsigned)win[buf][lane + 32 * r].x <= (unsigned)A.zero_row, "bwd gathered row");
        __syncwarp();
        if constexpr (RECOMP) {
            // the segment's records in one round trip: lane t fetches those of window entries t, t + 32
            // (padding entries: the all-zero record) and stages them for the batches below
            uint4 rc[NW];
#pragma unroll
            for (int r = 0; r < NW; ++r) rc[r] = __ldg(A.drec + win[buf][lane + 32 * r].x);
#pragma unroll
            for (int r = 0; r < NW; ++r) rec[lane + 32 * r] = rc[r];
            __syncwarp();
        }
        const float4 ai = ais[buf][q];
        float4 dacc = f4zero();
        float gsum[NW];
#pragma unroll
        for (int r = 0; r < NW; ++r) gsum[r] = 0.f;
#pragma unroll
        for (int b0 = 0; b0 < NB; b0 += RB) {
            if (b0 * EB < n) {
#pragma unroll
                for (int b = b0; b < b0 + RB; ++b)
                    if (b * EB < n)
                        bwd_batch<CB, HAS_DPREV, RECOMP>(A.d_out, win[buf] + b * EB, red + (b - b0) * EB * S, n - b * EB,
                                                         ai, g, q, dacc, pg, rec + b * EB, R);
                __syncwarp();
                // window entry e = lane + 32 r of this round: fixed-order sum of its G lane partials
#if !SMLP_EXP_NO_SDDMM
#pragma unroll
                for (int r = 0; r < NW; ++r) {
                    const int e = lane + 32 * r - b0 * EB;
                    if (e >= 0 && e < RB * EB && e + b0 * EB < n) {
                        const float* pr = red + e * S;
                        float t;
                        if constexpr (G % 4 == 0) {
                            float4 a4 = *reinterpret_cast<const float4*>(pr);
                            t = (a4.x + a4.y) + (a4.z + a4.w);
#pragma unroll
                            for (int v = 4; v < G; v += 4) {
                                a4 = *reinterpret_cast<const float4*>(pr + v);
                                t += (a4.x + a4.y) + (a4.z + a4.w);
                            }
                        } else {
                            t = pr[0];
#pragma unroll
                            for (int v = 1; v < G; ++v) t += pr[v];
                        }
                        gsum[r] = t;
                    }
                }
#endif
                __syncwarp();
            }
        }
        // gradient accumulation on the lane's own entries (coalesced)
#pragma unroll
        for (int r = 0; r < NW; ++r) {
            const int e = lane + 32 * r;
            if (e < n) st_hint(A.grad + cur.y + e, gsum[r] + gold[r], ps);
        }
        if (HAS_DPREV) {
            if (cur.w < 0) {
                float d[NR];
                group_reduce_scatter<CB>(dacc, g, d);
#if !SMLP_EXP_NO_EPI
                bwd_rows_epilogue<CB>(A, cur.x, d, sd, fp.off >> 2, lane);
#else
                if (lane == 0 && d[0] == 12345.f) A.d_prev[cur.x] = 0.f;
#endif
            } else {
                dacc = group_allreduce<G>(dacc);
                if (g == 0) st4(A.ws + (int64_t)cur.w * CB + q * 4, dacc);
            }
        }
        __syncwarp();
        cur = nxt;
        nxt = nn;
        buf ^= 1;
    }
}

template <int CB, int CBF, bool HAS_DPREV, bool GOLD, bool DROP>
__global__ void __launch_bounds__(256, 4) bwd_rows_kernel(BwdArgs A) {
    SMLP_PDL_ENTRY();
    __shared__ BwdRowsSmem<CB> sm;
    bwd_rows_body<CB, CBF, HAS_DPREV, GOLD, DROP>(A, hw_grid(), sm);
}
// the same with the implicit delta_l (layer L-1 under a dense-capped 2-output layer, no dropout)
template <int CB, int CBF, bool GOLD>
__global__ void __launch_bounds__(256, 4) bwd_rows_recomp_kernel(BwdArgs A) {
    SMLP_PDL_ENTRY();
    __shared__ BwdRowsSmem<CB> sm;
    __shared__ BwdRecSmem rsm;
    bwd_rows_body<CB, CBF, true, GOLD, false, true>(A, hw_grid(), sm, &rsm);
}

// ------------------------------------------------------------------------------------------
// narrow output layer (l = L, n_L <= NARROW_MAX): both passes walk the canonical CSR rows i of
// W^(L) in order, so a_{L-1} is streamed once instead of gathered once per output neuron.
// Lane t of a warp owns VEC = max(1, CB/32) consecutive batch columns; a warp takes RU rows at
// a time (all loads first, then the math) to keep enough bytes in flight.  The row's <= n_L
// entries sit one per lane; the weight of output jj is fetched by ballot + shuffle.
//   fwd: per-warp partial logits acc[jj][cols] -> per-CTA fixed-order sum -> the last CTA to
//        finish sums the CTA partials in CTA order and adds b_L (deterministic, no float atomics)
//   bwd: delta_L chunk held in registers; delta_{L-1}[i] = (sum_jj w_ij delta_L[jj]) * f' * keep,
//        g_ij = warp-sum over the chunk's columns of a_{L-1}[i] delta_L[j], Eq. 1 update of the
//        row's entries (coalesced), bias gradient of layer L-1
// ------------------------------------------------------------------------------------------
struct NarrowArgs {
    const int32_t* row_ptr;
    const int32_t* col;
    float* val;
    float* mom;
    float* grad;
    const float* a_prev;      // fwd: chunk base [n_in][CBf]; bwd: base of forward chunk c CB / CBf
    float* a_out;             // fwd: chunk base [n_out][CBf] (logits)
    const float* bias;        // fwd: b_L
    float* ws;                // fwd: [gridDim][NOUT][CB] CTA partials
    const float* d_out;       // bwd: delta_L chunk base [n_out][CB]
    float* d_prev;            // bwd: delta_{L-1} chunk base [n_in][CB]
    const uint4* zmask_prev;  // bwd: base of forward chunk c CB / CBf
    const uint4* kmask_prev;
    float* bgs;
    float* bias_prev;
    float* bias_mom_prev;
    float* bias_grad_prev;
    int64_t n_in;
    int n_out;
    int ncols;                // fwd: columns present in this launch (<= its width)
    const LayerMeta* meta;    // device nnz: complete layer (nnz = n_in n_out) -> row i = [i n_out, (i+1) n_out)
    uint4* drec;              // bwd, 2-output dense-capped layer: per-row record for the implicit delta_{L-1} (or null)
    float neg_slope_prev;
    float keep_scale_prev;
    int dropout_prev;
    int first, last;
    int fused;
    float lr, mu, wd;
};

template <int VEC>
__device__ __forceinline__ void ldvec(float (&d)[VEC], const float* p) {
    if constexpr (VEC == 4) {
        const float4 t = ldg4(p);
        d[0] = t.x; d[1] = t.y; d[2] = t.z; d[3] = t.w;
    } else if constexpr (VEC == 2) {
        const float2 t = __ldg(reinterpret_cast<const float2*>(p));
        d[0] = t.x; d[1] = t.y;
    } else {
        d[0] = __ldg(p);
    }
}

template <int VEC>
__device__ __forceinline__ void stvec(float* p, const float (&d)[VEC]) {
    if constexpr (VEC == 4) {
        *reinterpret_cast<float4*>(p) = make_float4(d[0], d[1], d[2], d[3]);
    } else if constexpr (VEC == 2) {
        *reinterpret_cast<float2*>(p) = make_float2(d[0], d[1]);
    } else {
        p[0] = d[0];
    }
}


// Row bounds of canonical row i: a dense-capped narrow layer has exactly n_out entries per row at
// i * n_out (no dependent row_ptr load on the critical path).
__device__ __forceinline__ void narrow_row(const NarrowArgs& A, bool dense, int64_t i, int& beg, int& len) {
    if (dense) {
        beg = (int)(i * A.n_out);
        len = A.n_out;
    } else {
        beg = __ldg(A.row_ptr + i);
        len = __ldg(A.row_ptr + i + 1) - beg;
    }
}

// The forward covers CB / CBF consecutive forward chunks per launch (CB columns, A.ncols of them
// present): one pass over the rows and weights for all of them; column b of the launch is column
// b % CBF of chunk b / CBF (FwdPos).  Each column's sum runs over the same rows in the same order
// whatever CB, so the logits do not depend on it.
template <int CB, int NOUT>
struct FwdNarrowSmem {
    float red[NOUT * CB];
};
template <int CB, int CBF, int NOUT>
__device__ __forceinline__ void fwd_narrow_body(const NarrowArgs& A, const VGrid vg, FwdNarrowSmem<CB, NOUT>& sm) {
    constexpr int VEC = CB >= 32 ? CB / 32 : 1;
    constexpr int RU = VEC == 4 ? 4 : 8;
    float* red = sm.red;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool colok = lane * VEC < A.ncols;
    const FwdPos<CB, CBF> fp(colok ? lane * VEC : 0, A.n_in);
    const int64_t r0 = (A.n_in * vg.bx) / vg.gx, r1 = (A.n_in * (vg.bx + 1)) / vg.gx;
    const bool dense = (int64_t)A.meta->nnz == A.n_in * (int64_t)A.n_out;   // graph-stable (device count)
    float acc[NOUT][VEC];
#pragma unroll
    for (int jj = 0; jj < NOUT; ++jj)
#pragma unroll
        for (int v = 0; v < VEC; ++v) acc[jj][v] = 0.f;
    for (int64_t i0 = r0 + (int64_t)warp * RU; i0 < r1; i0 += (int64_t)NARROW_WARPS * RU) {
        int cj[RU];
        float w[RU], a[RU][VEC];
        // all loads of the RU rows first (independent for dense rows), then the math
#pragma unroll
        for (int r = 0; r < RU; ++r) {
            const int64_t i = i0 + r;
            cj[r] = -1;
            w[r] = 0.f;
#pragma unroll
            for (int v = 0; v < VEC; ++v) a[r][v] = 0.f;
            if (i < r1) {
                int beg, len;
                narrow_row(A, dense, i, beg, len);
                if (lane < len) {
                    cj[r] = __ldg(A.col + beg + lane);
                    w[r] = A.val[beg + lane];
                }
                if (colok) ldvec<VEC>(a[r], A.a_prev + i * CBF + fp.aoff);
            }
        }
#pragma unroll
        for (int r = 0; r < RU; ++r) {
#pragma unroll
            for (int jj = 0; jj < NOUT; ++jj) {
                if (jj < A.n_out) {
                    const unsigned m = __ballot_sync(FULL, cj[r] == jj);
                    if (m) {
                        const float wj = __shfl_sync(FULL, w[r], __ffs(m) - 1);
#pragma unroll
                        for (int v = 0; v < VEC; ++v) acc[jj][v] = fmaf(wj, a[r][v], acc[jj][v]);
                    }
                }
            }
        }
    }
    // per-CTA fixed-order reduction over the warps: ((w0 + w1) + w2) + ...
    for (int wv = 0; wv < NARROW_WARPS; ++wv) {
        if (warp == wv && colok) {
#pragma unroll
            for (int jj = 0; jj < NOUT; ++jj)
#pragma unroll
                for (int v = 0; v < VEC; ++v) {
                    float& r = red[jj * CB + lane * VEC + v];
                    r = wv == 0 ? acc[jj][v] : r + acc[jj][v];
                }
        }
        __syncthreads();
    }
    for (int e = threadIdx.x; e < NOUT * CB; e += blockDim.x) A.ws[(int64_t)vg.bx * NOUT * CB + e] = red[e];
}
template <int CB, int CBF, int NOUT>
__global__ void __launch_bounds__(NARROW_WARPS * 32) fwd_narrow_kernel(NarrowArgs A) {
    SMLP_PDL_ENTRY();
    __shared__ FwdNarrowSmem<CB, NOUT> sm;
    fwd_narrow_body<CB, CBF, NOUT>(A, hw_grid(), sm);
}

// one warp per logit element e = jj * CB + b: fixed-order sum of the CTA partials (lane-strided,
// then an xor tree) + b_L, stored at column b % CBF of forward chunk b / CBF
template <int CB, int CBF, int NOUT>
__device__ __forceinline__ void fwd_narrow_finish_body(const NarrowArgs& A, int nparts, int e, int lane) {
    if (e % CB >= A.ncols) return;
    // lane b sums parts b, b + 32, ... in order; the loads of 8 parts are issued together (one
    // latency per 8 parts instead of one per part)
    float s = 0.f;
    for (int b0 = lane; b0 < nparts; b0 += 32 * 8) {
        float p[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int b = b0 + 32 * u;
            p[u] = b < nparts ? __ldg(A.ws + (int64_t)b * NOUT * CB + e) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) s += p[u];
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
    if (lane == 0) {
        const int jj = e / CB, b = e % CB;
        A.a_out[((int64_t)(b / CBF) * A.n_out + jj) * CBF + b % CBF] = s + __ldg(A.bias + jj);
    }
}
template <int CB, int CBF, int NOUT>
__global__ void __launch_bounds__(32) fwd_narrow_finish_kernel(NarrowArgs A, int nparts) {
    SMLP_PDL_ENTRY();
    fwd_narrow_finish_body<CB, CBF, NOUT>(A, nparts, blockIdx.x, threadIdx.x);
}

template <int CB, int CBF, int NOUT>
__global__ void __launch_bounds__(NARROW_WARPS * 32) bwd_narrow_kernel(NarrowArgs A) {
    SMLP_PDL_ENTRY();
    constexpr int VEC = CB >= 32 ? CB / 32 : 1;
    constexpr int RU = VEC == 4 ? 2 : (VEC == 2 ? 4 : 8);
    const int lane = threadIdx.x & 31;
    const bool colok = lane * VEC < CB;
    const FwdPos<CB, CBF> fp(colok ? lane * VEC : 0, A.n_in);   // the lane's columns, forward layout
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const bool dense = (int64_t)A.meta->nnz == A.n_in * (int64_t)A.n_out;   // graph-stable (device count)
    float dL[NOUT][VEC];
#pragma unroll
    for (int jj = 0; jj < NOUT; ++jj) {
#pragma unroll
        for (int v = 0; v < VEC; ++v) dL[jj][v] = 0.f;
        if (jj < A.n_out && colok) ldvec<VEC>(dL[jj], A.d_out + jj * CB + lane * VEC);
    }
    for (int64_t i0 = gw * RU; i0 < A.n_in; i0 += nw * RU) {
        int cj[RU], beg[RU];
        float w[RU], gacc[RU], a[RU][VEC];
        uint4 zb[RU], kb[RU];
        // all loads of the RU rows first (independent for dense rows), then the math
#pragma unroll
        for (int r = 0; r < RU; ++r) {
            const int64_t i = i0 + r;
            cj[r] = -1;
            w[r] = 0.f;
            gacc[r] = 0.f;
            beg[r] = 0;
            zb[r] = make_uint4(0, 0, 0, 0);
            kb[r] = make_uint4(FULL, FULL, FULL, FULL);
#pragma unroll
            for (int v = 0; v < VEC; ++v) a[r][v] = 0.f;
            if (i < A.n_in) {
                int len;
                narrow_row(A, dense, i, beg[r], len);
                if (lane < len) {
                    cj[r] = __ldg(A.col + beg[r] + lane);
                    w[r] = A.val[beg[r] + lane];
                    if (!A.first) gacc[r] = A.grad[beg[r] + lane];
                }
                if (colok) ldvec<VEC>(a[r], A.a_prev + i * CBF + fp.aoff);
                if (A.d_prev && colok) {
                    zb[r] = __ldg(A.zmask_prev + fp.moff + i);
                    if (A.dropout_prev) kb[r] = __ldg(A.kmask_prev + fp.moff + i);
                }
            }
        }
#pragma unroll
        for (int r = 0; r < RU; ++r) {
            const int64_t i = i0 + r;
            float dp[VEC];
#pragma unroll
            for (int v = 0; v < VEC; ++v) dp[v] = 0.f;
            float gmine = 0.f;
#pragma unroll
            for (int jj = 0; jj < NOUT; ++jj) {
                if (jj < A.n_out) {
                    const unsigned m = __ballot_sync(FULL, cj[r] == jj);
                    if (m) {
                        const float wj = __shfl_sync(FULL, w[r], __ffs(m) - 1);
                        float s = 0.f;
#pragma unroll
                        for (int v = 0; v < VEC; ++v) {
                            dp[v] = fmaf(wj, dL[jj][v], dp[v]);
                            s = fmaf(a[r][v], dL[jj][v], s);
                        }
#pragma unroll
                        for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
                        if (cj[r] == jj) gmine = s;
                    }
                }
            }
            if (i >= A.n_in) continue;   // warp-uniform
            if (cj[r] >= 0) {             // lane owns entry k = beg + lane: accumulate / apply Eq. 1
                const int64_t k = beg[r] + lane;
                const float gk = gmine + gacc[r];
                A.grad[k] = gk;
            }
            if (A.d_prev) {
                float o[VEC];
                float bsum = 0.f;
#pragma unroll
                for (int v = 0; v < VEC; ++v) {
                    const int b = fp.off + v;           // column within its forward chunk
                    const bool pos = (word(zb[r], b & 3) >> (b >> 2)) & 1u;
                    const bool keep = (word(kb[r], b & 3) >> (b >> 2)) & 1u;
                    const float x = dp[v] * (pos ? 1.f : A.neg_slope_prev);
                    o[v] = colok ? (A.dropout_prev ? (keep ? x * A.keep_scale_prev : 0.f) : x) : 0.f;
                    bsum += o[v];
                }
                if (colok) stvec<VEC>(A.d_prev + i * CB + lane * VEC, o);
#pragma unroll
                for (int off = 16; off >= 1; off >>= 1) bsum += __shfl_xor_sync(FULL, bsum, off);
                if (lane == 0) {
                    float tot = bsum;
                    if (!A.first) tot += A.bgs[i];
                    if (!A.last) A.bgs[i] = tot;
                    else A.bias_grad_prev[i] = tot;
                }
            }
        }
    }
}

// Narrow DENSE-CAPPED output layer, backward with one lane per canonical row i (32 rows per warp
// tile): the row's <= 16 weights, old gradients and masks sit in the lane's registers, the
// activation rows are staged through a per-warp shared-memory transpose (coalesced 16-B loads,
// conflict-free 16-B reads with a 36-float row stride) and delta_{L-1} goes back the same way.
// delta_L (n_L x CB) is broadcast from shared memory.  Rows of a dense-capped layer are either
// complete (j = 0..n_L-1 in order) or empty (outgoing row of a pruned neuron), so entry jj of a
// row is output jj.  ~10 warp instructions per row instead of ~200 with one row per warp.
template <int CB, int NOUT>
struct BwdNarrowRowsSmem {
    static constexpr int CS = CB < 32 ? CB : 32;     // columns per slice
    static constexpr int TS = CS + 1;                // odd smem row stride: lane-per-row access is conflict-free
    float dLs[NOUT][CB];
    float tile[NARROW_WARPS][32][TS];
};
template <int CB, int CBF, int NOUT>
__device__ __forceinline__ void bwd_narrow_rows_body(const NarrowArgs& A, const VGrid vg,
                                                     BwdNarrowRowsSmem<CB, NOUT>& sm) {
    constexpr int CS = CB < 32 ? CB : 32;     // columns per slice
    constexpr int NS = CB / CS;
    static_assert(CBF % CS == 0, "a slice lies inside one forward chunk");
    constexpr int TS = CS + 1;                // odd smem row stride: lane-per-row access is conflict-free
    constexpr int C4 = CS / 4;                // float4 per row slice
    auto& dLs = sm.dLs;
    auto& tile = sm.tile;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    for (int e = threadIdx.x; e < NOUT * CB; e += blockDim.x)
        dLs[e / CB][e % CB] = (e / CB < A.n_out) ? __ldg(A.d_out + e) : 0.f;
    __syncthreads();
    const uint64_t pol_s = policy_evict_first();
    const bool dense = (int64_t)A.meta->nnz == A.n_in * (int64_t)A.n_out;
    const int64_t ntiles = (A.n_in + 31) / 32;
    float* tl = &tile[wib][0][0];
    for (int64_t t = (int64_t)vg.bx * NARROW_WARPS + wib; t < ntiles; t += (int64_t)vg.gx * NARROW_WARPS) {
        const int64_t r0 = t * 32, i = r0 + lane;
        const bool valid = i < A.n_in;
        int beg = 0, len = 0;
        if (valid) narrow_row(A, dense, i, beg, len);
        float w[NOUT], gacc[NOUT], g[NOUT];
#pragma unroll
        for (int jj = 0; jj < NOUT; ++jj) {
            const bool has = jj < len;
            w[jj] = has ? ldrw_f32(A.val + beg + jj, pol_s) : 0.f;
            gacc[jj] = (has && !A.first) ? ldrw_f32(A.grad + beg + jj, pol_s) : 0.f;
            g[jj] = 0.f;
        }
        uint4 zb = make_uint4(0, 0, 0, 0), kb = make_uint4(FULL, FULL, FULL, FULL);
        float bsum = 0.f;
        uint32_t pw0 = 0u, pw1 = 0u;              // sign bits of the chunk's columns 0..31 / 32..63 (implicit delta record)
        for (int sl = 0; sl < NS; ++sl) {
            // a slice lies inside one forward chunk (CBF >= min(CB, 32) = CS): its rows and masks
            const FwdPos<CB, CBF> fp(sl * CS, A.n_in);
            if (A.d_prev && valid && fp.off == 0) {   // first slice of a forward chunk
                zb = __ldg(A.zmask_prev + fp.moff + i);
                if (A.dropout_prev) kb = __ldg(A.kmask_prev + fp.moff + i);
            }
#pragma unroll
            for (int m = 0; m < C4; ++m) {        // coalesced: 32 rows x CS columns of a_{L-1}
                const int e = lane + 32 * m, rr = e / C4, cc = e % C4;
                const int64_t row = r0 + rr;
                const float4 v = row < A.n_in
                                     ? ldro_f4(A.a_prev + row * CBF + fp.aoff + 4 * cc, pol_s)
                                     : f4zero();
                float* d = tl + rr * TS + 4 * cc;
                d[0] = v.x; d[1] = v.y; d[2] = v.z; d[3] = v.w;
            }
            __syncwarp();
#pragma unroll 4
            for (int c = 0; c < CS; ++c) {
                const int b = sl * CS + c;
                const float av = tl[lane * TS + c];
                float dp = 0.f;
#pragma unroll
                for (int jj = 0; jj < NOUT; ++jj) {
                    const float d = dLs[jj][b];
                    dp = fmaf(w[jj], d, dp);              // delta_L W^(L)T, outputs in order
                    g[jj] = fmaf(av, d, g[jj]);           // SDDMM over the chunk's columns
                }
                if (A.d_prev) {
                    const int bf = fp.off + c;            // column within its forward chunk
                    const bool pos = (word(zb, bf & 3) >> (bf >> 2)) & 1u;
                    const bool keep = (word(kb, bf & 3) >> (bf >> 2)) & 1u;
                    const float x = dp * (pos ? 1.f : A.neg_slope_prev);
                    const float o = A.dropout_prev ? (keep ? x * A.keep_scale_prev : 0.f) : x;
                    bsum += o;
                    tl[lane * TS + c] = o;
                    if constexpr (NOUT == 2 && CB <= 64) {
                        const uint32_t bit = (pos ? 1u : 0u) << (b & 31);
                        if (b & 32) pw1 |= bit;
                        else pw0 |= bit;
                    }
                }
            }
            __syncwarp();
            if (A.d_prev) {
#pragma unroll
                for (int m = 0; m < C4; ++m) {    // coalesced store of delta_{L-1}
                    const int e = lane + 32 * m, rr = e / C4, cc = e % C4;
                    const int64_t row = r0 + rr;
                    const float* d = tl + rr * TS + 4 * cc;
                    if (row < A.n_in) st4(A.d_prev + row * CB + sl * CS + 4 * cc, make_float4(d[0], d[1], d[2], d[3]));
                }
                __syncwarp();
            }
        }
        if (!valid) continue;
        if constexpr (NOUT == 2 && CB <= 64) {
            // implicit delta_{L-1}: the backward of W^(L-1) recomputes delta_{L-1}[i] of this chunk from
            // (sign bits, w_i0, w_i1) and delta_L with the very expression above
            if (A.drec) A.drec[i] = make_uint4(pw0, pw1, __float_as_uint(w[0]), __float_as_uint(w[1]));
        }
#pragma unroll
        for (int jj = 0; jj < NOUT; ++jj) {       // Eq. 1 / gradient accumulation of the row's entries
            if (jj < len) {
                const int64_t k = beg + jj;
                const float gk = g[jj] + gacc[jj];
                st_f32(A.grad + k, gk, pol_s);
            }
        }
        if (A.d_prev) {                           // bias gradient of layer L-1, accumulated over chunks
            float tot = bsum;
            if (!A.first) tot += A.bgs[i];
            if (!A.last) A.bgs[i] = tot;
            else A.bias_grad_prev[i] = tot;
        }
    }
}
template <int CB, int CBF, int NOUT>
__global__ void __launch_bounds__(NARROW_WARPS * 32) bwd_narrow_rows_kernel(NarrowArgs A) {
    SMLP_PDL_ENTRY();
    __shared__ BwdNarrowRowsSmem<CB, NOUT> sm;
    bwd_narrow_rows_body<CB, CBF, NOUT>(A, hw_grid(), sm);
}

// ------------------------------------------------------------------------------------------
// binary-input path of the first weight layer W^(2) (C5's inputs are {0,1}, stored fp32).
// When every staged input value is 0 or 1 (a device flag set by stage_input, so no host sync),
// a_1[b, i] is one bit and layer 2 needs no activation gather at all: the bit-packed input
// (16 B per input neuron for B <= 128, 1 MB for n_1 = 65536) is L1/L2-resident.  The result is
// bit-identical to the fp32 gather path: fmaf(w, x, acc) with x in {0, 1} in the same order.
//   fwd_bits: one warp per mirror row j covering ALL batch columns (lane q owns global columns
//             4q..4q+3 = chunk 4q/CB); epilogue as fwd_epilogue with group g = chunk g.
//   bwd_bits: one warp per mirror row j: delta_2[j] (all columns) in registers; per entry
//             g_ij = sum_b bit(b) delta_2[b, j] by a 32-entry transpose reduction, scattered to
//             the canonical grad slot mperm[t]; the Eq. 1 update then runs in canonical order.
// The fp32 chunk kernels of layer 2 return at once when the flag says binary, and these kernels
// return at once when it does not.
// ------------------------------------------------------------------------------------------
struct BitsArgs {
    const uint32_t* xbits;    // [n_1][XBITS_WORDS]
    const int32_t* nonbinary; // device flag
    int32_t* err;             // SMLP_INPUT_BINARY: set bit 2 when the batch is not binary (else null)
    const int32_t* mrow_ptr;
    const int32_t* msrc;
    const int32_t* mperm;
    const float* mval;
    const float* bias;
    float* a_out;             // act[2] base (all chunks)
    uint4* zmask;             // zmask[2] base
    uint4* kmask;
    const float* d_out;       // delta[2] base (all chunks)
    float* grad;              // canonical grad slice of W^(2)
    float* gmirror;           // [cap] gradient of W^(2) in mirror order (bwd_bits output)
    int64_t n_out;
    int nchunks;
    float neg_slope;
    int dropout_on;
    uint32_t drop_thr;
    float keep_scale;
    uint64_t seed;
    int rank;
    uint32_t step_lo;
    const uint64_t* step_ptr;
};

// Work unit of the bits kernels: BITS_ROWS consecutive mirror rows, streamed as one contiguous
// entry range in blocks of 32 entries (no per-row index latency; row ends come from the row
// pointers loaded once per unit).  Per block, lane t loads entry t's (src, w) (coalesced) and the
// 16-B bit row of its input neuron, and publishes (w, word k) pairs in shared memory; every lane
// then reads, per entry, the one pair holding its 4 columns' bits (broadcast, conflict-free).
constexpr int BITS_ROWS = 32;

struct FwdBitsSmem {
    float2 rec[WARPS_PER_BLOCK][32][XBITS_WORDS];
};
template <int CB, bool DROP>
__device__ __forceinline__ void fwd_bits_body(const BitsArgs& A, const VGrid vg, FwdBitsSmem& sm) {
    constexpr int G = CB / 4;                       // lanes per chunk
    auto& rec = sm.rec;
    if (*A.nonbinary) {
        if (A.err && vg.bx == 0 && threadIdx.x == 0) atomicOr(A.err, 2);   // promise broken
        return;
    }
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int g = lane / G, q = lane % G;            // chunk g, chunk-local lane q
    const bool colok = g < A.nchunks;
    const int wsel = lane >> 3, sh = (lane * 4) & 31;
    const uint32_t step_lo = A.step_ptr ? (uint32_t)(*A.step_ptr) : A.step_lo;
    const int64_t warp = ((int64_t)vg.bx * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)vg.gx * blockDim.x) >> 5;
    const int64_t nunits = (A.n_out + BITS_ROWS - 1) / BITS_ROWS;
    const uint4* xb4 = reinterpret_cast<const uint4*>(A.xbits);
    const float2* myrec = &rec[wib][0][wsel];
    for (int64_t u0 = warp; u0 < nunits; u0 += nwarps) {
        const int64_t j0 = u0 * BITS_ROWS;
        const int nrows = (int)(A.n_out - j0 < BITS_ROWS ? A.n_out - j0 : BITS_ROWS);
        const int rp_l = __ldg(A.mrow_ptr + j0 + min(lane, nrows));       // lane t: start of local row t
        const float b_l = lane < nrows ? __ldg(A.bias + j0 + lane) : 0.f;  // lane t: bias of local row t
        const int E0 = __shfl_sync(FULL, rp_l, 0), E1 = __ldg(A.mrow_ptr + j0 + nrows);
        int row = 0;
        int row_end = nrows > 1 ? __shfl_sync(FULL, rp_l, 1) : E1;
        float4 acc = f4zero();
        auto finish_row = [&]() {
            const int64_t j = j0 + row;
            const float bj = __shfl_sync(FULL, b_l, row);
            const float4 z = make_float4(acc.x + bj, acc.y + bj, acc.z + bj, acc.w + bj);
            uint32_t zb[4], kb[4];
            float out[4];
            // dropout (R13): one Philox block per (neuron j, batch rows 4 lane .. 4 lane + 3)
            uint4 dr = make_uint4(0, 0, 0, 0);
            if (DROP) dr = rng_stream(A.seed, P_DROPOUT, A.rank, 2, step_lo, ((uint64_t)j << 32) | (uint64_t)lane);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const float zc = comp(z, c);
                const bool pos = zc > 0.f;
                zb[c] = group_bits<G>(__ballot_sync(FULL, colok && pos), g);
                float a = pos ? zc : A.neg_slope * zc;
                bool keep = true;
                if (DROP) {
                    keep = word(dr, c) >= A.drop_thr;
                    a = keep ? a * A.keep_scale : 0.f;
                    kb[c] = group_bits<G>(__ballot_sync(FULL, colok && keep), g);
                }
                out[c] = a;
            }
            if (colok) {
                st4(A.a_out + ((int64_t)g * A.n_out + j) * CB + q * 4, make_float4(out[0], out[1], out[2], out[3]));
                if (q == 0) {
                    A.zmask[(int64_t)g * A.n_out + j] = make_uint4(zb[0], zb[1], zb[2], zb[3]);
                    if (DROP) A.kmask[(int64_t)g * A.n_out + j] = make_uint4(kb[0], kb[1], kb[2], kb[3]);
                }
            }
            acc = f4zero();
            ++row;
            row_end = __shfl_sync(FULL, rp_l, min(row + 1, 31));
            if (row + 1 > 31) row_end = E1;
        };
        // pipeline: (src, w) two blocks ahead, the 16-B bit row of each entry one block ahead
        auto ld_entry = [&](int k, int& sr, float& wv) {
            sr = k < E1 ? __ldg(A.msrc + k) : 0;
            wv = k < E1 ? __ldg(A.mval + k) : 0.f;
        };
        int src, src_n;
        float w, w_n;
        ld_entry(E0 + lane, src, w);
        ld_entry(E0 + 32 + lane, src_n, w_n);
        uint4 xb = E0 + lane < E1 ? __ldg(xb4 + src) : make_uint4(0, 0, 0, 0);
        for (int blk = E0; blk < E1; blk += 32) {
            int src_nn;
            float w_nn;
            ld_entry(blk + 64 + lane, src_nn, w_nn);
            const uint4 xb_n = blk + 32 + lane < E1 ? __ldg(xb4 + src_n) : make_uint4(0, 0, 0, 0);
            rec[wib][lane][0] = make_float2(w, __uint_as_float(__funnelshift_l(xb.x, xb.x, 1)));
            rec[wib][lane][1] = make_float2(w, __uint_as_float(__funnelshift_l(xb.y, xb.y, 1)));
            rec[wib][lane][2] = make_float2(w, __uint_as_float(__funnelshift_l(xb.z, xb.z, 1)));
            rec[wib][lane][3] = make_float2(w, __uint_as_float(__funnelshift_l(xb.w, xb.w, 1)));
            __syncwarp();
            const int n = min(32, E1 - blk);
            // the block's entries row by row: a tight loop up to the next row end, then the row's
            // epilogue (warp-uniform; empty rows finish at once)
            int u = 0;
            for (;;) {
                while (blk + u == row_end && row < nrows) finish_row();
                if (u >= n) break;
                const int stop = min(n, row_end - blk);
                const char* rp = reinterpret_cast<const char*>(myrec);
#pragma unroll 4
                for (; u < stop; ++u) {
                    const float2 r = *reinterpret_cast<const float2*>(rp + u * (XBITS_WORDS * 8));
                    // x in {0, 1}: acc + w x is acc + w for x = 1 and acc for x = 0, bit for bit, so
                    // each column is one predicated add.  The published word is rotated left by
                    // one: the lane's nibble lands on bits 1..4 and all four predicates come from
                    // one register-to-predicate move (R2P): 7 instructions per entry (LDS, SHF,
                    // R2P, 4 FADD) instead of ~18 with selects + FFMA2 (294 -> 216 us at C5)
                    const uint32_t rw = __float_as_uint(r.y);
                    const uint32_t nib = __funnelshift_r(rw, rw, sh);
                    if (nib & 2u) acc.x += r.x;
                    if (nib & 4u) acc.y += r.x;
                    if (nib & 8u) acc.z += r.x;
                    if (nib & 16u) acc.w += r.x;
                }
            }
            __syncwarp();
            w = w_n;
            src_n = src_nn;
            w_n = w_nn;
            xb = xb_n;
        }
        while (row < nrows) finish_row();
    }
}
template <int CB, bool DROP>
__global__ void __launch_bounds__(256) fwd_bits_kernel(BitsArgs A) {
    SMLP_PDL_ENTRY();
    __shared__ FwdBitsSmem sm;
    fwd_bits_body<CB, DROP>(A, hw_grid(), sm);
}


// Backward of the binary-input layer, one lane per mirror entry (i -> j): since x[b, i] is 0 or 1,
// g_ij = sum_b x[b, i] delta_2[b, j] is the sum of delta_2[b, j] over the SET bits b of input
// neuron i (5% of the batch at C5), added in ascending b (a fixed order).  The warp stages the
// row's delta_2[:, j] (<= 128 values, 4 chunks of CB) in shared memory once per output row j, and
// each lane walks its entry's 128-bit input row with ffs.  ~6 dependent adds per entry instead
// of 128 bit tests.  Rows are contiguous per warp; the next row's delta and entries are
// prefetched.  Output: the gradient in mirror order (gmirror), moved to the canonical order by
// grad_from_mirror_kernel.
struct BwdBitsSmem {
    __align__(16) float dsm_all[WARPS_PER_BLOCK][2][32 * XBITS_WORDS];
};
template <int CB>
__device__ __forceinline__ void bwd_bits_rows_body(const BitsArgs& A, const VGrid vg, BwdBitsSmem& sm) {
    if (*A.nonbinary) return;
    const int lane = threadIdx.x & 31;
    float (*dsm)[32 * XBITS_WORDS] = sm.dsm_all[threadIdx.x >> 5];
    const int64_t warp = ((int64_t)vg.bx * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)vg.gx * blockDim.x) >> 5;
    const int64_t r_lo = warp * A.n_out / nwarps, r_hi = (warp + 1) * A.n_out / nwarps;
    if (r_lo >= r_hi) return;
    const uint4* xb4 = reinterpret_cast<const uint4*>(A.xbits);
    // lane t stages columns 4t..4t+3 (chunk 4t / CB); columns past the batch are 0
    const int col = 4 * lane, chunk = col / CB;
    const bool colok = chunk < A.nchunks;
    auto dload = [&](int64_t j) -> float4 {
        return (colok && j < r_hi) ? ldg4(A.d_out + ((int64_t)chunk * A.n_out + j) * CB + (col % CB)) : f4zero();
    };
    int beg = A.mrow_ptr[r_lo];
    int end = A.mrow_ptr[r_lo + 1];
    int end_n = r_lo + 1 < r_hi ? A.mrow_ptr[r_lo + 2] : end;
    float4 d = dload(r_lo);
    int src = beg + lane < end ? __ldg(A.msrc + beg + lane) : 0;
    uint4 xb = beg + lane < end ? __ldg(xb4 + src) : make_uint4(0, 0, 0, 0);
    int buf = 0;
    for (int64_t j = r_lo; j < r_hi; ++j) {
        // prefetch the next row: delta column, first 32 entries and their bit rows
        const int end_nn = j + 2 < r_hi ? A.mrow_ptr[j + 3] : end_n;
        const float4 d_n = dload(j + 1);
        const int src_n = end + lane < end_n ? __ldg(A.msrc + end + lane) : 0;
        *reinterpret_cast<float4*>(&dsm[buf][col]) = d;
        __syncwarp();
        for (int base = beg; base < end; base += 32) {
            if (base != beg) {                                      // rows longer than 32
                src = base + lane < end ? __ldg(A.msrc + base + lane) : 0;
                xb = base + lane < end ? __ldg(xb4 + src) : make_uint4(0, 0, 0, 0);
            }
            float acc = 0.f;
#pragma unroll
            for (int c = 0; c < XBITS_WORDS; ++c) {
                uint32_t m = c == 0 ? xb.x : (c == 1 ? xb.y : (c == 2 ? xb.z : xb.w));
                while (m) {
                    acc += dsm[buf][c * 32 + __ffs(m) - 1];
                    m &= m - 1u;
                }
            }
            if (base + lane < end) A.gmirror[base + lane] = acc;
        }
        const uint4 xb_n = end + lane < end_n ? __ldg(xb4 + src_n) : make_uint4(0, 0, 0, 0);
        beg = end;
        end = end_n;
        end_n = end_nn;
        d = d_n;
        src = src_n;
        xb = xb_n;
        buf ^= 1;
    }
}

template <int CB>
__global__ void __launch_bounds__(256) bwd_bits_rows_kernel(BitsArgs A) {
    SMLP_PDL_ENTRY();
    __shared__ BwdBitsSmem sm;
    bwd_bits_rows_body<CB>(A, hw_grid(), sm);
}

// W^(2) gradient from mirror order to the canonical order of the grad view (a gather; a scatter
// would cost a sector read-fill)
struct MirrorGradArgs {
    const int32_t* nonbinary;
    const float* gm;
    const int32_t* minv;
    float* grad;
    const LayerMeta* meta;
};
__device__ __forceinline__ void grad_from_mirror_body(const MirrorGradArgs& M, const VGrid vg) {
    if (*M.nonbinary) return;
    const int64_t n = M.meta->nnz;
    for (int64_t k = (int64_t)vg.bx * blockDim.x + threadIdx.x; k < n; k += (int64_t)vg.gx * blockDim.x)
        M.grad[k] = __ldcg(M.gm + __ldg(M.minv + k));   // L2: gm was written by the previous phase
}
__global__ void grad_from_mirror_kernel(MirrorGradArgs M) {
    SMLP_PDL_ENTRY();
    grad_from_mirror_body(M, hw_grid());
}

// ------------------------------------------------------------------------------------------
// a6 standalone: Eq. 1 over the whole grad view (K > 1 path), then the mirror refresh
// ------------------------------------------------------------------------------------------
// Eq. 1 over one parameter slice (lam = weight decay, 0 for biases), 4 parameters per thread and
// two float4 groups in flight per iteration.  g and v are streamed once (evict_first); w is kept
// (evict_last): the mirror gather of the same layer reads it right after.
// G2: the fused path's split last-chunk gradient is in g2 (the update adds g2 + g)
struct UpdateArgs {
    float* w;
    float* v;
    const float* g;
    const float* g2;
    int64_t n;
    float lr, mu, wd;
    int64_t decay_end;
    float gs;
};
template <bool G2>
__device__ __forceinline__ void sgd_update4_body(const UpdateArgs& U, const VGrid vg) {
    float* __restrict__ w = U.w;
    float* __restrict__ v = U.v;
    const float* __restrict__ g = U.g;
    const float* __restrict__ g2 = U.g2;
    const int64_t n = U.n, decay_end = U.decay_end;
    const float lr = U.lr, mu = U.mu, wd = U.wd, gs = U.gs;
    const uint64_t pf = policy_evict_first(), pl = policy_evict_last();
    const int64_t n4 = n >> 2;
    const int64_t tid = (int64_t)vg.bx * blockDim.x + threadIdx.x, stride = (int64_t)vg.gx * blockDim.x;
    // weight decay on [0, decay_end) (the weight slices), none on the biases after it; decay_end
    // is a multiple of 32, so a float4 group never straddles it
    auto upd = [&](float4 wk, float4 vk, float4 gk, int64_t k4) {
        const float lam = 4 * k4 < decay_end ? wd : 0.f;
        float4 o;
        o.x = mu * vk.x - lr * (gs * gk.x + lam * wk.x);
        o.y = mu * vk.y - lr * (gs * gk.y + lam * wk.y);
        o.z = mu * vk.z - lr * (gs * gk.z + lam * wk.z);
        o.w = mu * vk.w - lr * (gs * gk.w + lam * wk.w);
        return o;
    };
    // the gradient: g, or (split last chunk) g2 + g = the last chunk's partial + the earlier
    // chunks' sum, the same two operands the in-kernel accumulation adds
    auto gload = [&](int64_t k4) {
        float4 a = ldg4_hint(g + 4 * k4, pf);
        if (G2) {
            const float4 b = ldg4_hint(g2 + 4 * k4, pf);
            a = make_float4(b.x + a.x, b.y + a.y, b.z + a.z, b.w + a.w);
        }
        return a;
    };
    int64_t k = tid;
    for (; k + stride < n4; k += 2 * stride) {
        const int64_t k2 = k + stride;
        const float4 w0 = ld4_hint(w + 4 * k, pl), v0 = ld4_hint(v + 4 * k, pf), g0 = gload(k);
        const float4 w1 = ld4_hint(w + 4 * k2, pl), v1 = ld4_hint(v + 4 * k2, pf), g1 = gload(k2);
        const float4 a = upd(w0, v0, g0, k), b = upd(w1, v1, g1, k2);
        const float4 wa = make_float4(w0.x + a.x, w0.y + a.y, w0.z + a.z, w0.w + a.w);
        const float4 wb = make_float4(w1.x + b.x, w1.y + b.y, w1.z + b.z, w1.w + b.w);
        st4_hint(v + 4 * k, a, pf);
        st4_hint(w + 4 * k, wa, pl);
        st4_hint(v + 4 * k2, b, pf);
        st4_hint(w + 4 * k2, wb, pl);
    }
    if (k < n4) {
        const float4 w0 = ld4_hint(w + 4 * k, pl), v0 = ld4_hint(v + 4 * k, pf), g0 = gload(k);
        const float4 a = upd(w0, v0, g0, k);
        const float4 wa = make_float4(w0.x + a.x, w0.y + a.y, w0.z + a.z, w0.w + a.w);
        st4_hint(v + 4 * k, a, pf);
        st4_hint(w + 4 * k, wa, pl);
    }
    if (tid < n - 4 * n4) {   // tail (n % 4 parameters)
        const int64_t t = 4 * n4 + tid;
        const float lam = t < decay_end ? wd : 0.f;
        const float gt = G2 ? g2[t] + g[t] : g[t];
        const float wk = w[t], vk = mu * v[t] - lr * (gs * gt + lam * wk);
        v[t] = vk;
        w[t] = wk + vk;
    }
}
template <bool G2>
__global__ void __launch_bounds__(256) sgd_update4_kernel(UpdateArgs U) {
    SMLP_PDL_ENTRY();
    sgd_update4_body<G2>(U, hw_grid());
}

// mirror refresh of several layers in one launch (small models: launch count matters more than
// overlap); blockIdx.y = layer
struct MirrorSet {
    const float* val[SMLP_MAX_LAYERS];
    const int32_t* mperm[SMLP_MAX_LAYERS];
    const LayerMeta* meta[SMLP_MAX_LAYERS];
    float* mval[SMLP_MAX_LAYERS];
};
__device__ __forceinline__ void mirror_values_multi_body(const MirrorSet& M, const VGrid vg) {
    const int l = vg.by;
    const int64_t n = M.meta[l]->nnz;
    for (int64_t t = (int64_t)vg.bx * blockDim.x + threadIdx.x; t < n; t += (int64_t)vg.gx * blockDim.x)
        M.mval[l][t] = __ldcg(M.val[l] + __ldg(M.mperm[l] + t));   // L2: val was just updated (persistent step)
}
__global__ void __launch_bounds__(256) mirror_values_multi_kernel(const __grid_constant__ MirrorSet M) {
    SMLP_PDL_ENTRY();
    mirror_values_multi_body(M, hw_grid());
}

// mirror copy mval[t] = val[mperm[t]], 4 consecutive t per thread (4 independent gathers in flight)
__global__ void __launch_bounds__(256) mirror_values_kernel(const float* __restrict__ val, const int32_t* __restrict__ mperm,
                                                            const LayerMeta* __restrict__ meta, float* __restrict__ mval) {
    SMLP_PDL_ENTRY();
    const uint64_t pf = policy_evict_first();
    const int64_t n = meta->nnz, n4 = n >> 2;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = tid; t < n4; t += stride) {
        const int4 p = ldi4_hint(mperm + 4 * t, pf);
        st4_hint(mval + 4 * t, make_float4(__ldg(val + p.x), __ldg(val + p.y), __ldg(val + p.z), __ldg(val + p.w)), pf);
    }
    if (tid < n - 4 * n4) mval[4 * n4 + tid] = __ldg(val + __ldg(mperm + 4 * n4 + tid));
}

// Short-row backward (128-column chunks, canonical rows averaging < 8 entries: the eps = 1
// widths), the counterpart of fwd_short_rows_kernel: a warp streams 32 consecutive canonical rows
// as one entry range (col, w, row id loaded coalesced per 32-entry block), gathers 4 entries'
// delta_l[j] rows and a_{l-1}[i] rows at a time across row boundaries; per entry the SDDMM
// partial is summed over the 32 lanes by a fixed butterfly and kept by lane (entry mod 32) for
// one coalesced gradient store per block; delta_{l-1} rows are accumulated in entry order and
// finished (bwd_rows_epilogue) as each row's last entry is added, with the rows' mask bits and
// bias data loaded once per unit (lane t = row t).  No Eq. 1 in-kernel (the fused path's UPD
// variant keeps the row kernel).
template <bool HAS_DPREV, bool GOLD, bool DROP>
__global__ void __launch_bounds__(256, 4) bwd_short_rows_kernel(BwdArgs A) {
    SMLP_PDL_ENTRY();
    constexpr int CB = 128, GU = 4, NR = RowCfg<CB>::NR;
    __shared__ int4 rec_all[WARPS_PER_BLOCK][32 + GU];
    if (A.skip_if_binary && *A.skip_if_binary == 0) return;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    int4* rec = rec_all[wib];
    const uint64_t pg = gather_policy(A.l2hint), ps = stream_policy(A.l2hint);
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t nunits = (A.n_prev + SHORT_ROWS - 1) / SHORT_ROWS;
    for (int64_t u0 = warp; u0 < nunits; u0 += nwarps) {
        const int64_t i0 = u0 * SHORT_ROWS;
        const int nrows = (int)(A.n_prev - i0 < SHORT_ROWS ? A.n_prev - i0 : SHORT_ROWS);
        const int rp_l = __ldg(A.row_ptr + i0 + min(lane, nrows));
        const int E0 = __shfl_sync(FULL, rp_l, 0), E1 = __ldg(A.row_ptr + i0 + nrows);
        if (lane < GU) rec[32 + lane] = make_int4(A.zero_row, 0, (int)i0, 0);   // padding: zero delta row
        // the unit's rows' epilogue side data, lane t = row t (loaded once, shuffled at the finish)
        uint4 zb_l = make_uint4(0, 0, 0, 0), kb_l = make_uint4(FULL, FULL, FULL, FULL);
        float bgs_l = 0.f;
        if (HAS_DPREV && lane < nrows) {
            zb_l = A.zmask_prev[i0 + lane];
            if (DROP) kb_l = A.kmask_prev[i0 + lane];
            if (!A.first) bgs_l = A.bgs[i0 + lane];
        }
        int row = 0;
        int row_end = nrows > 1 ? __shfl_sync(FULL, rp_l, 1) : E1;
        float4 dacc = f4zero();
        auto finish_rows_at = [&](int e) {
            while (row < nrows && e == row_end) {
                if (HAS_DPREV) {
                    BwdSide sd;
                    sd.zb = make_uint4(__shfl_sync(FULL, zb_l.x, row), __shfl_sync(FULL, zb_l.y, row),
                                       __shfl_sync(FULL, zb_l.z, row), __shfl_sync(FULL, zb_l.w, row));
                    sd.kb = DROP ? make_uint4(__shfl_sync(FULL, kb_l.x, row), __shfl_sync(FULL, kb_l.y, row),
                                              __shfl_sync(FULL, kb_l.z, row), __shfl_sync(FULL, kb_l.w, row))
                                 : make_uint4(FULL, FULL, FULL, FULL);
                    sd.bgs = __shfl_sync(FULL, bgs_l, row);
                    const float d[NR] = {dacc.x, dacc.y, dacc.z, dacc.w};
                    bwd_rows_epilogue<CB>(A, i0 + row, d, sd, lane, lane);
                }
                dacc = f4zero();
                ++row;
                row_end = row + 1 < nrows ? __shfl_sync(FULL, rp_l, min(row + 1, 31)) : E1;
            }
        };
        for (int blk = E0; blk < E1; blk += 32) {
            const int n = min(32, E1 - blk);
            __syncwarp();
            if (lane < n) {
                const int k = blk + lane;
                rec[lane] = make_int4(ld_hint_i(A.col + k, ps), __float_as_int(ld_hint(A.val + k, ps)),
                                      ld_hint_i(A.rowid + k, ps), 0);
            } else {
                rec[lane] = make_int4(A.zero_row, 0, (int)i0, 0);
            }
            SMLP_BOUND((unsigned)rec[lane].x <= (unsigned)A.zero_row, "bwd short gathered row");
            const float gold_l = GOLD && lane < n ? ld_hint(A.grad + blk + lane, ps) : 0.f;
            __syncwarp();
            float gval = 0.f;                              // lane t: the SDDMM gradient of entry t
            for (int v0 = 0; v0 < n; v0 += GU) {
                float4 x[GU], a[GU];
                float wv[GU];
#pragma unroll
                for (int k = 0; k < GU; ++k) {
                    const int4 e = rec[v0 + k];
                    wv[k] = __int_as_float(e.y);
                    x[k] = ldg4_hint(A.d_out + (int64_t)e.x * CB + lane * 4, pg);
                    a[k] = ldg4_hint(A.a_prev + (int64_t)e.z * CB + lane * 4, ps);
                }
#pragma unroll
                for (int k = 0; k < GU; ++k) {             // g = <a_{l-1}[i], delta_l[j]>, fixed butterfly
                    float p = dot4p(a[k], x[k]);
#pragma unroll
                    for (int m = 16; m >= 1; m >>= 1) p += __shfl_xor_sync(FULL, p, m);
                    if (lane == v0 + k) gval = p;
                }
                if (HAS_DPREV) {                           // delta_{l-1} rows, one row segment at a time
                    const int kmax = min(GU, n - v0);
                    int k = 0;
                    for (;;) {
                        finish_rows_at(blk + v0 + k);
                        if (k >= kmax) break;
                        const int stop = min(kmax, row_end - (blk + v0));
#pragma unroll
                        for (int kk = 0; kk < GU; ++kk)
                            if (kk >= k && kk < stop) fma4p(dacc, wv[kk], x[kk]);
                        k = stop;
                    }
                }
            }
            if (lane < n) st_hint(A.grad + blk + lane, gval + gold_l, ps);
        }
        if (HAS_DPREV) finish_rows_at(E1);
    }
}

// ==========================================================================================
// Persistent step (small models; DESIGN.md §5 "persistent step").  A model of <= 4M parameters
// is launch- and latency-bound: its ~17 kernels per step each do a few microseconds of work.  For
// such a model every API call (forward; backward + Eq. 1 + mirror refresh) is ONE cooperative
// launch of persist_step_kernel: one resident wave of 256-thread blocks that runs the call's
// kernels as phases -- the same __device__ bodies the standalone kernels run, with the same
// virtual grids, so the results are bit-identical -- separated by grid-wide barriers.  The phase
// list is recorded by the host code that would otherwise launch the kernels (Recorder below) and
// passed by value as the kernel parameter.
// ==========================================================================================
enum PhaseKind : int {
    PK_STAGE = 0, PK_FWD_ROWS, PK_FWD_FINISH, PK_FWD_NARROW, PK_FWD_NARROW_FIN, PK_SOFTMAX,
    PK_BWD_ROWS, PK_BWD_FINISH, PK_BWD_NARROW_ROWS, PK_UPDATE, PK_MIRROR, PK_RESET_FLAG, PK_FWD_BITS, PK_BWD_BITS,
    PK_GRAD_FROM_MIRROR
};
constexpr int PMAX = 24;
union PhaseArgs {
    StageArgs st;
    FwdArgs f;
    NarrowArgs n;
    SoftmaxArgs s;
    BwdArgs b;
    UpdateArgs u;
    BitsArgs bits;
    MirrorGradArgs mg;
    int32_t* flag;
};
struct PPhase {
    int kind;
    int gx, gy;   // virtual grid (PK_FWD_NARROW_FIN: gx = CTA partials, gy = logit elements)
    int sub;      // PK_FWD_NARROW*/PK_BWD_NARROW_ROWS: padded n_L; PK_BWD_ROWS: HAS_DPREV 4 | GOLD 2 | DROP 1
    PhaseArgs a;
};
struct PProgram {
    int n;
    int nsm;         // SMs of the device (each hosts exactly gridDim.x / nsm blocks of the wave)
    unsigned* bar;   // grid barrier state [count, generation] (the handle's, zeroed at create)
    unsigned* smslot;   // [nsm] blocks placed on each SM so far (the handle's; grows by the wave's share per launch)
    MirrorSet mirror;
    PPhase ph[PMAX];
};

template <int CB>
union PhaseSmem {
    FwdRowsSmem<CB> fr;
    BwdRowsSmem<CB> br;
    StageSmem st;
    SoftmaxSmem so;
    FwdNarrowSmem<CB, NARROW_MAX> fn;
    BwdNarrowRowsSmem<CB, 16> bn;
    FwdBitsSmem fb;
    BwdBitsSmem bb;
};
// the phase's arguments are copied from the kernel parameter into shared memory at the start of
// every phase (one coalesced read per block): the bodies read their fields from shared memory
// instead of through generic pointers into the parameter buffer (an L2 round trip after every
// barrier's L1 invalidation, several of them dependent per phase)
template <int CB>
struct PersistSmem {
    __align__(16) PhaseArgs args[2];   // double-buffered: phase i + 1's are loaded during phase i's barrier
    __align__(16) PhaseSmem<CB> u;
};
__device__ __forceinline__ void stage_phase_args(PhaseArgs& dst, const PhaseArgs& src, int t0) {
    const int* s = reinterpret_cast<const int*>(&src);
    int* d = reinterpret_cast<int*>(&dst);
    for (int w = (int)threadIdx.x - t0; w < (int)(sizeof(PhaseArgs) / sizeof(int)); w += (int)blockDim.x - t0)
        if (w >= 0) d[w] = s[w];
}

// Phase entry points of the persistent kernel: real (non-inlined) calls, so each phase body gets
// its own register allocation instead of sharing one with every other phase of the switch.  The
// arguments are read in place from the shared-memory copy the kernel staged (a private copy per
// thread measured 1.6x slower: the 250-500 B structs spill at 64 registers).
template <int CB>
__device__ __noinline__ void pk_stage(int bx, const StageArgs& S, int gx, int gy, PersistSmem<CB>& sm) {
    for (int v = bx; v < gx * gy; v += gridDim.x) {
        stage_input_body(S, VGrid{v % gx, v / gx, gx}, sm.u.st);
        __syncthreads();
    }
}
template <int CB>
__device__ __noinline__ void pk_fwd_rows(int bx, const FwdArgs& A, PersistSmem<CB>& sm) {
    fwd_rows_body<CB>(A, VGrid{bx, 0, (int)gridDim.x}, sm.u.fr);
}
template <int CB>
__device__ __noinline__ void pk_fwd_finish(int bx, const FwdArgs& A) {
    fwd_finish_body<CB>(A, VGrid{bx, 0, (int)gridDim.x});
}
template <int CB, int NOUT>
__device__ __noinline__ void pk_fwd_narrow(int bx, const NarrowArgs& A, int gx, PersistSmem<CB>& sm) {
    if constexpr (CB * NOUT <= NARROW_MAX_ELEMS) {
        for (int v = bx; v < gx; v += gridDim.x) {
            fwd_narrow_body<CB, CB, NOUT>(A, VGrid{v, 0, gx}, *reinterpret_cast<FwdNarrowSmem<CB, NOUT>*>(&sm.u));
            __syncthreads();
        }
    }
}
template <int CB, int NOUT>
__device__ __noinline__ void pk_fwd_narrow_fin(int bx, const NarrowArgs& A, int nparts, int count) {
    const int lane = threadIdx.x & 31;
    const int gw = (int)((bx * blockDim.x + threadIdx.x) >> 5), nw = (int)((gridDim.x * blockDim.x) >> 5);
    for (int e = gw; e < count; e += nw) fwd_narrow_finish_body<CB, CB, NOUT>(A, nparts, e, lane);
}
template <int CB, int NOUT>
__device__ __noinline__ void pk_bwd_narrow(int bx, const NarrowArgs& A, PersistSmem<CB>& sm) {
    if constexpr (CB * NOUT <= NARROW_MAX_ELEMS && NOUT <= 16)
        bwd_narrow_rows_body<CB, CB, NOUT>(A, VGrid{bx, 0, (int)gridDim.x},
                                           *reinterpret_cast<BwdNarrowRowsSmem<CB, NOUT>*>(&sm.u));
}
template <int CB, bool HD, bool GO, bool DR>
__device__ __noinline__ void pk_bwd_rows(int bx, const BwdArgs& A, PersistSmem<CB>& sm) {
    bwd_rows_body<CB, CB, HD, GO, DR>(A, VGrid{bx, 0, (int)gridDim.x}, sm.u.br);
}
template <int CB>
__device__ __noinline__ void pk_bwd_finish(int bx, const BwdArgs& A) {
    bwd_finish_body<CB, CB>(A, VGrid{bx, 0, (int)gridDim.x});
}
template <int CB>
__device__ __noinline__ void pk_softmax(int bx, const SoftmaxArgs& A, PersistSmem<CB>& sm) {
    if (bx == 0) softmax_ce_body(A, sm.u.so);
}
template <int CB, bool DROP>
__device__ __noinline__ void pk_fwd_bits(int bx, const BitsArgs& A, PersistSmem<CB>& sm) {
    fwd_bits_body<CB, DROP>(A, VGrid{bx, 0, (int)gridDim.x}, sm.u.fb);
}
template <int CB>
__device__ __noinline__ void pk_bwd_bits(int bx, const BitsArgs& A, PersistSmem<CB>& sm) {
    bwd_bits_rows_body<CB>(A, VGrid{bx, 0, (int)gridDim.x}, sm.u.bb);
}
__device__ __noinline__ void pk_grad_from_mirror(int bx, const MirrorGradArgs& M) {
    grad_from_mirror_body(M, VGrid{bx, 0, (int)gridDim.x});
}
__device__ __noinline__ void pk_update(int bx, const UpdateArgs& U) {
    sgd_update4_body<false>(U, VGrid{bx, 0, (int)gridDim.x});
}
__device__ __noinline__ void pk_mirror(int bx, const MirrorSet& M, int gx, int gy) {
    for (int v = bx; v < gx * gy; v += gridDim.x) mirror_values_multi_body(M, VGrid{v % gx, v / gx, gx});
}

// Grid-wide barrier of the persistent kernel (all blocks are co-resident: cooperative launch).
// One arrival atomic per block; the last arrival resets the count and bumps the generation word,
// the others poll it with volatile (L2) loads.  cg::this_grid().sync() polls with an L1
// invalidation per iteration (CCTL.IVALL), which -- with 4 blocks per SM still working on a phase
// -- wipes their L1 (spilled registers, gathered rows) thousands of times per barrier; measured
// 2.5x slower steps.  Here the L1 is invalidated once, by the acquire fence after the wait.
__device__ __forceinline__ void grid_barrier(unsigned* bar, PhaseArgs* next = nullptr, const PhaseArgs* next_src = nullptr) {
    __syncthreads();
    // warps 1..7 stage the next phase's arguments while thread 0 waits for the other blocks
    if (next && threadIdx.x >= 32) stage_phase_args(*next, *next_src, 32);
    if (threadIdx.x == 0) {
        volatile unsigned* gen_p = bar + 1;
        const unsigned gen = *gen_p;
        __threadfence();                                  // release this block's writes of the phase
        if (atomicAdd(bar, 1u) == gridDim.x - 1) {
            atomicExch(bar, 0u);
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (*gen_p == gen) __nanosleep(20);
        }
        __threadfence();                                  // acquire: later loads see every block's writes
    }
    __syncthreads();
}

#ifdef SMLP_PERSIST_TIMING
__device__ unsigned long long g_phase_ns[PMAX + 1];
#endif
template <int CB>
__global__ void __launch_bounds__(256, 4) persist_step_kernel(const __grid_constant__ PProgram P) {
#ifdef SMLP_PERSIST_TIMING
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_phase_ns[PMAX] = t;
    }
#endif
    extern __shared__ __align__(16) unsigned char psm_raw[];
    PersistSmem<CB>& sm = *reinterpret_cast<PersistSmem<CB>*>(psm_raw);
    // Spread block index: a cooperative wave places CONSECUTIVE blocks on the same few SMs
    // (measured: blocks 0-23 of 592 on SMs 142-147, tools/smid_probe.cu), so a phase with few
    // virtual blocks (staging, the narrow output layer, softmax) would run on 1-6 SMs.  Each
    // block takes slot k of its SM instead; bx = k * nsm + smid is a permutation of the grid in
    // which bx = 0 .. nsm-1 sit on distinct SMs.  (Every SM hosts exactly gridDim.x / nsm blocks;
    // the counters are cleared at the end of the launch.)
    __shared__ int s_bx;
    if (threadIdx.x == 0) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        const unsigned per_sm = gridDim.x / (unsigned)P.nsm;
        const unsigned slot = atomicAdd(P.smslot + smid, 1u) % per_sm;
        s_bx = (int)(slot * (unsigned)P.nsm + smid);
    }
    __syncthreads();
    const int bx = s_bx;
    if (P.n > 0) stage_phase_args(sm.args[0], P.ph[0].a, 0);
    __syncthreads();
    for (int i = 0; i < P.n; ++i) {
        const PPhase& ph = P.ph[i];
        const int nout = ph.sub;
        const PhaseArgs& a = sm.args[i & 1];
        // a finish phase with no split rows (device counts, the same in every block) is skipped
        // together with its barrier
        if ((ph.kind == PK_FWD_FINISH && a.f.meta->n_fmulti == 0) ||
            (ph.kind == PK_BWD_FINISH && a.b.meta->n_bmulti == 0)) {
            // (skipped with its barrier; the next phase's arguments go to the other buffer now)
            if (i + 1 < P.n) stage_phase_args(sm.args[(i + 1) & 1], P.ph[i + 1].a, 0);
            __syncthreads();
            continue;
        }
        switch (ph.kind) {
            case PK_STAGE: pk_stage<CB>(bx, a.st, ph.gx, ph.gy, sm); break;
            case PK_FWD_ROWS: pk_fwd_rows<CB>(bx, a.f, sm); break;
            case PK_FWD_FINISH: pk_fwd_finish<CB>(bx, a.f); break;
            case PK_FWD_NARROW:
                if (nout == 2) pk_fwd_narrow<CB, 2>(bx, a.n, ph.gx, sm);
                else if (nout == 4) pk_fwd_narrow<CB, 4>(bx, a.n, ph.gx, sm);
                else if (nout == 8) pk_fwd_narrow<CB, 8>(bx, a.n, ph.gx, sm);
                else if (nout == 16) pk_fwd_narrow<CB, 16>(bx, a.n, ph.gx, sm);
                else pk_fwd_narrow<CB, 32>(bx, a.n, ph.gx, sm);
                break;
            case PK_FWD_NARROW_FIN:
                if (nout == 2) pk_fwd_narrow_fin<CB, 2>(bx, a.n, ph.gx, ph.gy);
                else if (nout == 4) pk_fwd_narrow_fin<CB, 4>(bx, a.n, ph.gx, ph.gy);
                else if (nout == 8) pk_fwd_narrow_fin<CB, 8>(bx, a.n, ph.gx, ph.gy);
                else if (nout == 16) pk_fwd_narrow_fin<CB, 16>(bx, a.n, ph.gx, ph.gy);
                else pk_fwd_narrow_fin<CB, 32>(bx, a.n, ph.gx, ph.gy);
                break;
            case PK_SOFTMAX: pk_softmax<CB>(bx, a.s, sm); break;
            case PK_BWD_ROWS:
                switch (ph.sub) {
                    case 4: pk_bwd_rows<CB, true, false, false>(bx, a.b, sm); break;
                    case 5: pk_bwd_rows<CB, true, false, true>(bx, a.b, sm); break;
                    case 6: pk_bwd_rows<CB, true, true, false>(bx, a.b, sm); break;
                    case 7: pk_bwd_rows<CB, true, true, true>(bx, a.b, sm); break;
                    case 0: pk_bwd_rows<CB, false, false, false>(bx, a.b, sm); break;
                    case 2: pk_bwd_rows<CB, false, true, false>(bx, a.b, sm); break;
                    default: break;
                }
                break;
            case PK_BWD_FINISH: pk_bwd_finish<CB>(bx, a.b); break;
            case PK_BWD_NARROW_ROWS:
                if (nout == 2) pk_bwd_narrow<CB, 2>(bx, a.n, sm);
                else if (nout == 4) pk_bwd_narrow<CB, 4>(bx, a.n, sm);
                else if (nout == 8) pk_bwd_narrow<CB, 8>(bx, a.n, sm);
                else pk_bwd_narrow<CB, 16>(bx, a.n, sm);
                break;
            case PK_UPDATE: pk_update(bx, a.u); break;
            case PK_MIRROR: pk_mirror(bx, P.mirror, ph.gx, ph.gy); break;
            case PK_RESET_FLAG:
                if (bx == 0 && threadIdx.x == 0) *a.flag = 0;
                break;
            case PK_FWD_BITS:
                if (ph.sub) pk_fwd_bits<CB, true>(bx, a.bits, sm);
                else pk_fwd_bits<CB, false>(bx, a.bits, sm);
                break;
            case PK_BWD_BITS: pk_bwd_bits<CB>(bx, a.bits, sm); break;
            case PK_GRAD_FROM_MIRROR: pk_grad_from_mirror(bx, a.mg); break;
            default: break;
        }
        // every phase's writes are visible to the next (and smem is free again)
        if (i + 1 < P.n) grid_barrier(P.bar, &sm.args[(i + 1) & 1], &P.ph[i + 1].a);
        else grid_barrier(P.bar);
#ifdef SMLP_PERSIST_TIMING    // A/B build only: per-phase end times (ns) after the barrier
        if (bx == 0 && threadIdx.x == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            g_phase_ns[i] = t;
        }
#endif
    }
    // every block took its slot before the first barrier: clear the counters for the next launch
    if (bx == 0)
        for (int t = threadIdx.x; t < P.nsm; t += blockDim.x) P.smslot[t] = 0;
}

// Host side: the launch sites record their phases here while h->rec is set (no launch, no count)
struct Recorder {
    PProgram P;
    bool ok = true;
    PPhase* add(int kind, int gx, int gy, int sub) {
        if (P.n >= PMAX) {
            ok = false;
            return nullptr;
        }
        PPhase* ph = &P.ph[P.n++];
        ph->kind = kind;
        ph->gx = gx;
        ph->gy = gy;
        ph->sub = sub;
        return ph;
    }
};
inline Recorder* recorder(smlp_handle* h) { return static_cast<Recorder*>(h->rec); }

// grid of the finish kernels: their row count lives in device memory (graph-stable), so the grid
// is sized for the capacity but capped at 2 blocks per SM (grid-stride loops): split rows are rare
// (C5: ~0.03% of the rows), and a wider grid of mostly idle blocks costs a few microseconds per launch
int persistent_grid(const smlp_handle* h, int64_t groups, int groups_per_warp) {
    const int64_t warps = (groups + groups_per_warp - 1) / groups_per_warp;
    const int64_t need = (warps + WARPS_PER_BLOCK - 1) / WARPS_PER_BLOCK;
    const int64_t cap = (int64_t)h->num_sms * 2;
    return (int)std::max<int64_t>(1, std::min(need, cap));
}

// one resident wave of a row kernel: blocks/SM from the occupancy calculator (cached per kernel)
template <typename K>
int rows_grid(const smlp_handle* h, K kernel, int64_t segs) {
    static int per_sm = 0;
    if (per_sm == 0) {
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, WARPS_PER_BLOCK * 32, 0) != cudaSuccess ||
            per_sm < 1)
            per_sm = 1;
    }
    const int64_t need = (segs + WARPS_PER_BLOCK - 1) / WARPS_PER_BLOCK;
    return (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)per_sm * h->num_sms));
}

// rows a layer needs for the streaming short-row kernels: one 32-row unit per resident warp
// (SMLP_SHORT_MIN_ROWS overrides, e.g. 0 for small parity tests)
static int64_t short_min_rows(const smlp_handle* h) {
    return h->short_min_rows >= 0 ? h->short_min_rows : (int64_t)SHORT_ROWS * 32 * h->num_sms;
}

template <int CB>
int launch_fwd(smlp_handle* h, const FwdArgs& A, const Layer& L) {
    constexpr int P = 32 / (CB / 4);
    if (Recorder* R = recorder(h)) {
        const bool short_rows = CB == 128 && L.nnz < (int64_t)h->short_max_fwd * L.n_out && L.n_out >= short_min_rows(h);
        if (CB != h->CB || short_rows) {
            R->ok = false;
            return SMLP_OK;
        }
        if (PPhase* ph = R->add(PK_FWD_ROWS, 0, 0, 0)) ph->a.f = A;
        if (L.fslot_cap > 0)
            if (PPhase* ph = R->add(PK_FWD_FINISH, 0, 0, 0)) ph->a.f = A;
        return SMLP_OK;
    }
    if constexpr (CB == 128) {
        // layers of short rows (< 16 entries per mirror row on average): stream whole rows
        // (and enough 32-row units to give every resident warp one: a narrow layer keeps the row kernel)
        if (L.nnz < (int64_t)h->short_max_fwd * L.n_out &&
            L.n_out >= short_min_rows(h)) {
            const int64_t units = (L.n_out + SHORT_ROWS - 1) / SHORT_ROWS;
            launch_pdl(h->pdl, fwd_short_rows_kernel, rows_grid(h, fwd_short_rows_kernel, units), WARPS_PER_BLOCK * 32, h->stream, A);
            SMLP_CK_LAUNCH(h, "fwd_short_rows_kernel");
            return SMLP_OK;
        }
    }
    launch_pdl(h->pdl, fwd_rows_kernel<CB>, rows_grid(h, fwd_rows_kernel<CB>, L.fseg_cap), WARPS_PER_BLOCK * 32, h->stream, A);
    SMLP_CK_LAUNCH(h, "fwd_rows_kernel");
    if (L.fslot_cap > 0) {
        const int g2 = persistent_grid(h, std::max<int64_t>(1, L.fslot_cap / 2), P);
        launch_pdl(h->pdl, fwd_finish_kernel<CB>, g2, WARPS_PER_BLOCK * 32, h->stream, A);
        SMLP_CK_LAUNCH(h, "fwd_finish_kernel");
    }
    return SMLP_OK;
}

template <int CB, int CBF>
int launch_bwd(smlp_handle* h, const BwdArgs& A, const Layer& L, bool has_dprev) {
    constexpr int P = 32 / (CB / 4);
    const bool gold = !A.first && !A.no_gold, drop = A.dropout_prev != 0;
    if (Recorder* R = recorder(h)) {
        const bool short_rows = CB == 128 && CBF == 128 && L.nnz < (int64_t)h->short_max_bwd * L.n_in &&
                                L.n_in >= short_min_rows(h);
        if (CB != CBF || CB != h->CB || short_rows) {
            R->ok = false;
            return SMLP_OK;
        }
        const int mode = (has_dprev ? 4 : 0) | (gold ? 2 : 0) | (drop ? 1 : 0);
        if (PPhase* ph = R->add(PK_BWD_ROWS, 0, 0, mode)) ph->a.b = A;
        if (has_dprev && L.bslot_cap > 0)
            if (PPhase* ph = R->add(PK_BWD_FINISH, 0, 0, 0)) ph->a.b = A;
        return SMLP_OK;
    }
    if constexpr (CB == 128 && CBF == 128) {
        // layers of short canonical rows (< 8 entries on average): stream whole rows
        if (L.nnz < (int64_t)h->short_max_bwd * L.n_in &&
            L.n_in >= short_min_rows(h)) {
            const int64_t units = (L.n_in + SHORT_ROWS - 1) / SHORT_ROWS;
#define SMLP_BWD_SHORT(HD, GO, DR)                                                                          \
    if (has_dprev == HD && gold == GO && drop == DR) {                                                    \
        launch_pdl(h->pdl, bwd_short_rows_kernel<HD, GO, DR>, rows_grid(h, bwd_short_rows_kernel<HD, GO, DR>, units), WARPS_PER_BLOCK * 32, h->stream, A); \
        SMLP_CK_LAUNCH(h, "bwd_short_rows_kernel");                                                       \
        return SMLP_OK;                                                                                   \
    }
            SMLP_BWD_SHORT(true, false, false)
            SMLP_BWD_SHORT(true, false, true)
            SMLP_BWD_SHORT(true, true, false)
            SMLP_BWD_SHORT(true, true, true)
            SMLP_BWD_SHORT(false, false, false)
            SMLP_BWD_SHORT(false, true, false)
#undef SMLP_BWD_SHORT
        }
    }
    if constexpr (CB <= 64) {
        if (A.drec) {   // implicit delta_l: records instead of delta rows (has_dprev, no dropout: api.cu)
            if (gold)
                launch_pdl(h->pdl, bwd_rows_recomp_kernel<CB, CBF, true>, rows_grid(h, bwd_rows_recomp_kernel<CB, CBF, true>, L.bseg_cap), WARPS_PER_BLOCK * 32, h->stream, A);
            else
                launch_pdl(h->pdl, bwd_rows_recomp_kernel<CB, CBF, false>, rows_grid(h, bwd_rows_recomp_kernel<CB, CBF, false>, L.bseg_cap), WARPS_PER_BLOCK * 32, h->stream, A);
            SMLP_CK_LAUNCH(h, "bwd_rows_recomp_kernel");
            if (L.bslot_cap > 0) {
                const int g2 = persistent_grid(h, std::max<int64_t>(1, L.bslot_cap / 2), P);
                launch_pdl(h->pdl, bwd_finish_kernel<CB, CBF>, g2, WARPS_PER_BLOCK * 32, h->stream, A);
                SMLP_CK_LAUNCH(h, "bwd_finish_kernel");
            }
            return SMLP_OK;
        }
    }
    const int mode = (has_dprev ? 4 : 0) | (gold ? 2 : 0) | (drop ? 1 : 0);
#define SMLP_BWD_ROWS(HD, GO, DR)                                                                             \
case (HD ? 4 : 0) | (GO ? 2 : 0) | (DR ? 1 : 0):                                                            \
    launch_pdl(h->pdl, bwd_rows_kernel<CB, CBF, HD, GO, DR>, rows_grid(h, bwd_rows_kernel<CB, CBF, HD, GO, DR>, L.bseg_cap), WARPS_PER_BLOCK * 32, h->stream, A); \
    break;
    switch (mode) {
        SMLP_BWD_ROWS(true, false, false)
        SMLP_BWD_ROWS(true, false, true)
        SMLP_BWD_ROWS(true, true, false)
        SMLP_BWD_ROWS(true, true, true)
        SMLP_BWD_ROWS(false, false, false)
        SMLP_BWD_ROWS(false, true, false)
        default: return set_err(h, SMLP_E_ARG, "bwd_rows_kernel: bad mode");
    }
#undef SMLP_BWD_ROWS
    SMLP_CK_LAUNCH(h, "bwd_rows_kernel");
    if (has_dprev && L.bslot_cap > 0) {
        const int g2 = persistent_grid(h, std::max<int64_t>(1, L.bslot_cap / 2), P);
        launch_pdl(h->pdl, bwd_finish_kernel<CB, CBF>, g2, WARPS_PER_BLOCK * 32, h->stream, A);
        SMLP_CK_LAUNCH(h, "bwd_finish_kernel");
    }
    return SMLP_OK;
}

#define SMLP_DISPATCH_CB(h, width, fn, ...)                            \
    switch (width) {                                                   \
        case 4: return fn<4>(__VA_ARGS__);                             \
        case 8: return fn<8>(__VA_ARGS__);                             \
        case 16: return fn<16>(__VA_ARGS__);                           \
        case 32: return fn<32>(__VA_ARGS__);                           \
        case 64: return fn<64>(__VA_ARGS__);                           \
        case 128: return fn<128>(__VA_ARGS__);                         \
        default: return set_err((h), SMLP_E_ARG, "unsupported chunk_batch"); \
    }

// backward kernels: (CB, CBf) pairs -- equal widths, or the forward tensors 2 / 4 times narrower
// (CBf >= 32, api.cu)
#define SMLP_DISPATCH_PAIR(h, cb, cbf, fn, ...)                                          \
    switch ((cb) * 1000 + (cbf)) {                                                       \
        case 4004: return fn<4, 4>(__VA_ARGS__);                                         \
        case 8008: return fn<8, 8>(__VA_ARGS__);                                         \
        case 16016: return fn<16, 16>(__VA_ARGS__);                                      \
        case 32032: return fn<32, 32>(__VA_ARGS__);                                      \
        case 64064: return fn<64, 64>(__VA_ARGS__);                                      \
        case 64032: return fn<64, 32>(__VA_ARGS__);                                      \
        case 128128: return fn<128, 128>(__VA_ARGS__);                                   \
        case 128064: return fn<128, 64>(__VA_ARGS__);                                    \
        case 128032: return fn<128, 32>(__VA_ARGS__);                                    \
        default: return set_err((h), SMLP_E_ARG, "unsupported (chunk_batch, forward chunk) pair"); \
    }

int dispatch_fwd(smlp_handle* h, const FwdArgs& A, const Layer& L) { SMLP_DISPATCH_CB(h, h->CBf, launch_fwd, h, A, L); }
int dispatch_bwd(smlp_handle* h, const BwdArgs& A, const Layer& L, bool hd) {
    SMLP_DISPATCH_PAIR(h, h->CB, h->CBf, launch_bwd, h, A, L, hd);
}

template <int CB, int CBF, int NOUT>
int launch_narrow_n(smlp_handle* h, const NarrowArgs& A, const Layer& L, bool fwd) {
    if constexpr (NOUT * CB > NARROW_MAX_ELEMS) {
        return set_err(h, SMLP_E_ARG, "narrow output layer too wide for chunk_batch");
    } else {
        if (Recorder* R = recorder(h)) {
            if (CB != CBF || CB != h->CB || (!fwd && !(NOUT <= 16 && L.dense))) {
                R->ok = false;
                return SMLP_OK;
            }
            if (fwd) {
                if (PPhase* ph = R->add(PK_FWD_NARROW, L.ngrid, 1, NOUT)) ph->a.n = A;
                if (PPhase* ph = R->add(PK_FWD_NARROW_FIN, L.ngrid, A.n_out * CB, NOUT)) ph->a.n = A;
            } else {
                if (PPhase* ph = R->add(PK_BWD_NARROW_ROWS, 0, 0, NOUT)) ph->a.n = A;
            }
            return SMLP_OK;
        }
        if (fwd) {
            launch_pdl(h->pdl, fwd_narrow_kernel<CB, CBF, NOUT>, L.ngrid, NARROW_WARPS * 32, h->stream, A);
            SMLP_CK_LAUNCH(h, "fwd_narrow_kernel");
            launch_pdl(h->pdl, fwd_narrow_finish_kernel<CB, CBF, NOUT>, A.n_out * CB, 32, h->stream, A, L.ngrid);
            SMLP_CK_LAUNCH(h, "fwd_narrow_finish_kernel");
        } else {
            if constexpr (NOUT <= 16) {
                if (L.dense) {
                    const int64_t tiles = (A.n_in + 31) / 32;
                    const int64_t blocks = std::min<int64_t>((tiles + NARROW_WARPS - 1) / NARROW_WARPS, (int64_t)h->num_sms * 4);
                    launch_pdl(h->pdl, bwd_narrow_rows_kernel<CB, CBF, NOUT>, (int)std::max<int64_t>(1, blocks), NARROW_WARPS * 32, h->stream, A);
                    SMLP_CK_LAUNCH(h, "bwd_narrow_rows_kernel");
                    return SMLP_OK;
                }
            }
            constexpr int VEC = CB >= 32 ? CB / 32 : 1;
            constexpr int RU = VEC == 4 ? 2 : (VEC == 2 ? 4 : 8);
            const int64_t warps = (A.n_in + RU - 1) / RU;
            const int64_t blocks = std::min<int64_t>((warps + NARROW_WARPS - 1) / NARROW_WARPS, (int64_t)h->num_sms * 3);
            launch_pdl(h->pdl, bwd_narrow_kernel<CB, CBF, NOUT>, (int)std::max<int64_t>(1, blocks), NARROW_WARPS * 32, h->stream, A);
            SMLP_CK_LAUNCH(h, "bwd_narrow_kernel");
        }
        return SMLP_OK;
    }
}

// forward: CB = the launch's width (a multiple of CBF = the forward width); backward: the (CB, CBf) pair
template <int CB, int CBF>
int launch_narrow(smlp_handle* h, const NarrowArgs& A, const Layer& L, bool fwd) {
    switch (L.nout_pad) {
        case 2: return launch_narrow_n<CB, CBF, 2>(h, A, L, fwd);
        case 4: return launch_narrow_n<CB, CBF, 4>(h, A, L, fwd);
        case 8: return launch_narrow_n<CB, CBF, 8>(h, A, L, fwd);
        case 16: return launch_narrow_n<CB, CBF, 16>(h, A, L, fwd);
        case 32: return launch_narrow_n<CB, CBF, 32>(h, A, L, fwd);
        default: return set_err(h, SMLP_E_ARG, "narrow layer: bad padded width");
    }
}
template <int CB, int CBF>
int launch_narrow_fwd(smlp_handle* h, const NarrowArgs& A, const Layer& L) { return launch_narrow<CB, CBF>(h, A, L, true); }
template <int CB, int CBF>
int launch_narrow_bwd(smlp_handle* h, const NarrowArgs& A, const Layer& L) { return launch_narrow<CB, CBF>(h, A, L, false); }

// fwd: `width` columns (CB / CBf forward chunks) per launch; bwd: one backward chunk
int dispatch_narrow(smlp_handle* h, const NarrowArgs& A, const Layer& L, bool fwd, int width) {
    if (fwd) {
        SMLP_DISPATCH_PAIR(h, width, h->CBf, launch_narrow_fwd, h, A, L);
    }
    SMLP_DISPATCH_PAIR(h, h->CB, h->CBf, launch_narrow_bwd, h, A, L);
}

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
    launch_pdl(h->pdl, mirror_values_kernel, launch_grid(h, (Ly.cap + 3) / 4, 256), 256, h->stream, Ly.val, Ly.mperm, Ly.meta, Ly.mval);
    SMLP_CK_LAUNCH(h, "mirror_values_kernel");
    return SMLP_OK;
}

int run_probs(smlp_handle* h, int B, float* probs) {
    if (Recorder* R = recorder(h)) {
        R->ok = false;
        return SMLP_OK;
    }
    launch_pdl(h->pdl, softmax_probs_kernel, (B + 127) / 128, 128, h->stream, h->act[h->L], probs, h->sizes[h->L - 1], B, h->CBf);
    SMLP_CK_LAUNCH(h, "softmax_probs_kernel");
    return SMLP_OK;
}

BitsArgs bits_args(smlp_handle* h, Layer& L2, int nchunks) {
    BitsArgs A{};
    A.xbits = h->xbits;
    A.nonbinary = h->d_nonbinary;
    A.err = h->input_binary ? h->d_err : nullptr;
    A.mrow_ptr = L2.mrow_ptr;
    A.msrc = L2.msrc;
    A.mperm = L2.mperm;
    A.mval = L2.mval;
    A.bias = L2.bias;
    A.a_out = h->act[2];
    A.zmask = h->zmask[2];
    A.kmask = h->kmask[2];
    A.d_out = h->delta[2];
    A.grad = L2.grad;
    A.gmirror = h->gmirror2;
    A.n_out = L2.n_out;
    A.nchunks = nchunks;
    A.neg_slope = neg_slope_of(h, 2);
    A.drop_thr = drop_threshold(h->dropout);
    A.keep_scale = (float)(1.0 / (1.0 - (double)h->dropout));
    A.seed = h->seed;
    A.rank = h->rank;
    A.step_ptr = h->step_counter;
    return A;
}

template <int CB>
int launch_bits(smlp_handle* h, const BitsArgs& A, const Layer& L2, bool fwd) {
    const int64_t units = (L2.n_out + BITS_ROWS - 1) / BITS_ROWS;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((units + WARPS_PER_BLOCK - 1) / WARPS_PER_BLOCK,
                                                                  (int64_t)h->num_sms * 6));
    if (fwd) {
        // units are grid-strided: one resident wave (blocks/SM from the occupancy calculator)
        if (A.dropout_on)
            launch_pdl(h->pdl, fwd_bits_kernel<CB, true>, rows_grid(h, fwd_bits_kernel<CB, true>, units), WARPS_PER_BLOCK * 32, h->stream, A);
        else
            launch_pdl(h->pdl, fwd_bits_kernel<CB, false>, rows_grid(h, fwd_bits_kernel<CB, false>, units), WARPS_PER_BLOCK * 32, h->stream, A);
        SMLP_CK_LAUNCH(h, "fwd_bits_kernel");
    } else {
        const int g2 = (int)std::max<int64_t>(1, std::min<int64_t>((L2.n_out + 8 * WARPS_PER_BLOCK - 1) /
                                                                     (8 * WARPS_PER_BLOCK),
                                                                 (int64_t)h->num_sms * 8));
        launch_pdl(h->pdl, bwd_bits_rows_kernel<CB>, g2, WARPS_PER_BLOCK * 32, h->stream, A);
        SMLP_CK_LAUNCH(h, "bwd_bits_rows_kernel");
    }
    return SMLP_OK;
}

int dispatch_bits(smlp_handle* h, const BitsArgs& A, const Layer& L2, bool fwd) {
    if (Recorder* R = recorder(h)) {
        if ((fwd ? h->CBf : h->CB) != h->CB) R->ok = false;
        else if (PPhase* ph = R->add(fwd ? PK_FWD_BITS : PK_BWD_BITS, 0, 0, A.dropout_on ? 1 : 0)) ph->a.bits = A;
        return SMLP_OK;
    }
    SMLP_DISPATCH_CB(h, fwd ? h->CBf : h->CB, launch_bits, h, A, L2, fwd);
}

// forward: chunk c of the forward layout; backward: a_{L-1} from forward chunk c CB / CBf (the
// backward chunk's first columns, FwdPos)
NarrowArgs narrow_args(smlp_handle* h, Layer& Ly, int c, bool fwd) {
    const int CB = h->CBf;
    const int fc = fwd ? c : c * (h->CB / h->CBf);
    const int64_t nin = Ly.n_in, nout = Ly.n_out;
    NarrowArgs A{};
    A.row_ptr = Ly.row_ptr;
    A.col = Ly.col;
    A.val = Ly.val;
    A.mom = Ly.mom;
    A.grad = Ly.grad;
    A.a_prev = h->act[Ly.l - 1] + (int64_t)fc * nin * CB;
    A.a_out = fwd ? h->act[Ly.l] + (int64_t)c * nout * CB : nullptr;
    A.bias = Ly.bias;
    A.ws = Ly.nws;
    A.n_in = nin;
    A.n_out = (int)nout;
    A.ncols = CB;
    A.meta = Ly.meta;
    return A;
}

static int run_forward_phases(smlp_handle* h, const float* x, const int32_t* x_idx, int B, bool train, uint64_t step,
                              float* probs) {
    const int CB = h->CBf;    // the forward tensors' chunk width
    const int nchunks = (B + CB - 1) / CB;
    {
        dim3 grid((unsigned)((h->sizes[0] + 127) / 128), (unsigned)((nchunks * CB + 31) / 32));
        const int vec = (h->sizes[0] % 4 == 0) && ((uintptr_t)x % 16 == 0);
        prof_start(h, K_STAGE, 1, 8.0 * (double)B * (double)h->sizes[0], 0.0);
        const StageArgs S{x, x_idx, B, nchunks, CB, h->sizes[0], h->act[1], h->xbits, h->d_nonbinary, vec};
        if (Recorder* R = recorder(h)) {
            if (h->xbits)                    // the non-binary flag is cleared one phase before staging sets it
                if (PPhase* ph = R->add(PK_RESET_FLAG, 1, 1, 0)) ph->a.flag = h->d_nonbinary;
            if (PPhase* ph = R->add(PK_STAGE, (int)grid.x, (int)grid.y, 0)) ph->a.st = S;
        } else {
            if (h->xbits) SMLP_CK(h, cudaMemsetAsync(h->d_nonbinary, 0, sizeof(int32_t), h->stream));
            launch_pdl(h->pdl, stage_input_kernel, grid, 256, h->stream, S);
            SMLP_CK_LAUNCH(h, "stage_input_kernel");
        }
        prof_stop(h);
    }
    const bool drop = train && h->dropout > 0.f;
    if (h->xbits) {   // binary-input layer 2, all chunks in one pass (returns at once if not binary)
        Layer& L2 = h->layers[0];
        BitsArgs A = bits_args(h, L2, nchunks);
        A.dropout_on = drop ? 1 : 0;
        A.step_lo = (uint32_t)step;
        prof_start(h, K_FWD_BITS, 2, 12.0 * (double)L2.nnz + 4.0 * B * (double)(L2.n_in + L2.n_out),
                   2.0 * (double)L2.nnz * B);
        SMLP_TRY(dispatch_bits(h, A, L2, true));
        prof_stop(h);
    }
    // chunk-major order: layer l+1 of chunk c gathers the slab layer l of chunk c just wrote,
    // while it is still in L2
    for (int c = 0; c < nchunks; ++c) {
        for (int l = 2; l <= h->L; ++l) {
            Layer& Ly = h->layers[l - 2];
            const int64_t nin = h->sizes[l - 2], nout = h->sizes[l - 1];
            const int Bc = std::min(CB, B - c * CB);
            const double nnz = (double)Ly.nnz;
            if (Ly.narrow) continue;   // after the chunk loop, several chunks per pass
            FwdArgs A{};
            A.a_prev = h->act[l - 1] + (int64_t)c * nin * CB;
            A.a_out = h->act[l] + (int64_t)c * nout * CB;
            const bool hidden = l < h->L;
            A.zmask = hidden ? h->zmask[l] + (int64_t)c * nout : nullptr;
            A.kmask = hidden ? h->kmask[l] + (int64_t)c * nout : nullptr;
            A.seg = Ly.fseg;
            A.multi = Ly.fmulti;
            A.mrow_ptr = Ly.mrow_ptr;
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
            A.skip_if_binary = (l == 2 && h->xbits) ? h->d_nonbinary : nullptr;
            A.zero_row = (int)((int64_t)(h->max_chunks_f - c) * nin);
            A.l2hint = 1;
            prof_start(h, K_FWD, l, 12.0 * nnz / nchunks + 4.0 * Bc * (double)(nin + nout), 2.0 * nnz * Bc);
            SMLP_TRY(dispatch_fwd(h, A, Ly));
            prof_stop(h);
        }
    }
    // narrow output layer: one pass over its rows and weights per W columns (W / CBf forward chunks;
    // the earlier chunks' a_{L-1} slabs come back from HBM, cheaper than one row pass per chunk)
    if (h->layers[h->L - 2].narrow) {
        Layer& Ly = h->layers[h->L - 2];
        const int64_t nin = Ly.n_in, nout = Ly.n_out;
        int W = CB;
        if (CB >= 32)
            while (W < 128 && W < nchunks * CB && (int64_t)Ly.nout_pad * W * 2 <= NARROW_MAX_ELEMS) W *= 2;
        for (int c = 0; c < nchunks; c += W / CB) {
            NarrowArgs A = narrow_args(h, Ly, c, true);
            A.ncols = std::min(W, (nchunks - c) * CB);
            const int Bc = std::min(A.ncols, B - c * CB);
            prof_start(h, K_FWD, h->L, 8.0 * (double)Ly.nnz + 4.0 * Bc * (double)(nin + nout),
                       2.0 * (double)Ly.nnz * Bc);
            SMLP_TRY(dispatch_narrow(h, A, Ly, true, W));
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

// Eq. 1 over the parameter slice [lo, hi) on `stream`: one resident wave (8 CTAs of 256 per SM),
// two float4 groups per thread and iteration
static int launch_update(smlp_handle* h, cudaStream_t stream, int64_t lo, int64_t hi, bool decay, const smlp_sgd* sgd,
                         bool g2 = false) {
    if (hi <= lo) return SMLP_OK;
    constexpr int threads = 256;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((hi - lo + 4 * threads - 1) / (4 * threads),
                                                                 (int64_t)h->num_sms * 8));
    // decay: weights (all of [lo, hi)), or none (biases), or -- for the single whole-view launch of
    // small models -- everything below bias_base
    const int64_t decay_end = decay ? std::min(hi, h->bias_base) - lo : 0;
    float* w = h->param + lo;
    float* v = h->mom + lo;
    const float* g = h->grad + lo;
    const float* gb = g2 ? h->grad2 + lo : nullptr;
    const UpdateArgs U{w, v, g, gb, hi - lo, sgd->lr, sgd->momentum, sgd->weight_decay, decay_end, sgd->grad_scale};
    if (Recorder* R = recorder(h)) {
        if (g2 || stream != h->stream) R->ok = false;
        else if (PPhase* ph = R->add(PK_UPDATE, 0, 0, 0)) ph->a.u = U;
        return SMLP_OK;
    }
    if (g2)
        launch_pdl(h->pdl, sgd_update4_kernel<true>, grid, threads, stream, U);
    else
        launch_pdl(h->pdl, sgd_update4_kernel<false>, grid, threads, stream, U);
    SMLP_CK_LAUNCH(h, "sgd_update4_kernel");
    return SMLP_OK;
}

static int ensure_aux(smlp_handle* h) {
    if (h->aux_stream) return SMLP_OK;
    SMLP_CK(h, cudaStreamCreateWithFlags(&h->aux_stream, cudaStreamNonBlocking));
    for (auto& e : h->aux_ev) SMLP_CK(h, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    return SMLP_OK;
}

// W^(l)'s gradient (and b_{l-1}'s) is final: record the layer event (sparse_mlp_wait_layer lets a
// communication stream start that layer's allreduce while the backward continues)
static int layer_done(smlp_handle* h, int l) {
    if (h->rec) return SMLP_OK;   // persistent step: recorded after its launch (every layer at once)
    if (!h->layer_ev[l]) SMLP_CK(h, cudaEventCreateWithFlags(&h->layer_ev[l], cudaEventDisableTiming));
    SMLP_CK(h, cudaEventRecord(h->layer_ev[l], h->stream));
    return SMLP_OK;
}

static int run_backward_phases(smlp_handle* h, const int32_t* labels, const int32_t* y_idx, float* loss,
                               bool split_last, const smlp_sgd* early = nullptr) {
    const int CB = h->CB;
    const int B = h->trace_B;
    const int nchunks = (B + CB - 1) / CB;
    const int L = h->L;
    for (auto& Ly : h->layers) Ly.updated_early = false;
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
        S.CBf = h->CBf;
        prof_start(h, K_SOFTMAX, L, 8.0 * (double)B * (double)S.nL, 0.0);
        if (Recorder* R = recorder(h)) {
            if (PPhase* ph = R->add(PK_SOFTMAX, 1, 1, 0)) ph->a.s = S;
        } else {
            launch_pdl(h->pdl, softmax_ce_kernel, 1, 256, h->stream, S);
            SMLP_CK_LAUNCH(h, "softmax_ce_kernel");
        }
        prof_stop(h);
    }
    // chunk-major, chunks in reverse: the forward ended on the last chunk, and layer l of chunk c
    // gathers the delta_l slab layer l+1 of chunk c just wrote (L2-resident).  Gradients
    // accumulate over the chunks in this fixed order.
    for (int c = nchunks - 1; c >= 0; --c) {
        const bool first = c == nchunks - 1, last = c == 0;
        for (int l = L; l >= 2; --l) {
            Layer& Ly = h->layers[l - 2];
            const int64_t nin = h->sizes[l - 2], nout = h->sizes[l - 1];
            const bool has_dprev = l >= 3;
            const int fc = c * (CB / h->CBf);                      // first forward chunk of chunk c
            Layer* Lp = has_dprev ? &h->layers[l - 3] : nullptr;   // owner of bias b_{l-1}
            const int Bc = std::min(CB, B - c * CB);
            const double nnz = (double)Ly.nnz;
            const double act_bytes = 4.0 * Bc * (double)(nin + nout + (has_dprev ? nin : 0));
            const int dropout_prev = (has_dprev && h->trace_train && h->dropout > 0.f) ? 1 : 0;
            const float keep_scale = (float)(1.0 / (1.0 - (double)h->dropout));
            if (Ly.narrow_bwd) {
                NarrowArgs A = narrow_args(h, Ly, c, false);
                A.d_out = h->delta[l] + (int64_t)c * nout * CB;
                A.d_prev = has_dprev ? h->delta[l - 1] + (int64_t)c * nin * CB : nullptr;
                A.zmask_prev = has_dprev ? h->zmask[l - 1] + (int64_t)fc * nin : nullptr;
                A.kmask_prev = has_dprev ? h->kmask[l - 1] + (int64_t)fc * nin : nullptr;
                A.bgs = Ly.bgs;
                A.bias_prev = Lp ? Lp->bias : nullptr;
                A.bias_mom_prev = Lp ? Lp->bias_mom : nullptr;
                A.bias_grad_prev = Lp ? Lp->bias_grad : nullptr;
                A.neg_slope_prev = neg_slope_of(h, l - 1);
                A.keep_scale_prev = keep_scale;
                A.dropout_prev = dropout_prev;
                A.first = first;
                A.last = last;
                A.drec = (l == L && has_dprev) ? h->drec : nullptr;
                prof_start(h, K_BWD, l, 12.0 * nnz / nchunks + act_bytes, (has_dprev ? 4.0 : 2.0) * nnz * Bc);
                SMLP_TRY(dispatch_narrow(h, A, Ly, false, CB));
                prof_stop(h);
                if (last) SMLP_TRY(layer_done(h, l));
                continue;
            }
            BwdArgs A{};
            A.a_prev = h->act[l - 1] + (int64_t)fc * nin * h->CBf;   // forward layout (FwdPos)
            A.d_out = h->delta[l] + (int64_t)c * nout * CB;
            A.d_prev = has_dprev ? h->delta[l - 1] + (int64_t)c * nin * CB : nullptr;
            A.zmask_prev = has_dprev ? h->zmask[l - 1] + (int64_t)fc * nin : nullptr;
            A.kmask_prev = has_dprev ? h->kmask[l - 1] + (int64_t)fc * nin : nullptr;
            A.n_prev = nin;
            A.row_ptr = Ly.row_ptr;
            A.rowid = Ly.rowid;
            A.seg = Ly.bseg;
            A.multi = Ly.bmulti;
            A.meta = Ly.meta;
            A.col = Ly.col;
            A.val = Ly.val;
            A.mom = Ly.mom;
            A.grad = Ly.grad;
            A.ws = Ly.bws;
            A.bgs = Ly.bgs;
            A.bias_prev = Lp ? Lp->bias : nullptr;
            A.bias_mom_prev = Lp ? Lp->bias_mom : nullptr;
            A.bias_grad_prev = Lp ? Lp->bias_grad : nullptr;
            A.neg_slope_prev = neg_slope_of(h, l - 1);
            A.dropout_prev = dropout_prev;
            A.keep_scale_prev = keep_scale;
            A.first = first;
            A.last = last;
            A.skip_if_binary = (l == 2 && h->xbits) ? h->d_nonbinary : nullptr;
            // the last of several chunks writes its gradient to grad2 instead of adding the earlier
            // chunks' sum (read back from grad); the Eq. 1 pass that follows adds the two
            // (W^(2) with the bit path keeps one buffer: its gradient may come from the bit kernels)
            Ly.split = false;
            if (split_last && last && !first && h->grad2 && !(l == 2 && h->xbits)) {
                A.grad = h->grad2 + Ly.val_off;
                A.no_gold = 1;
                Ly.split = true;
            }
            A.zero_row = (int)((int64_t)(h->max_chunks - c) * nout);
            A.l2hint = 1;
            if (l == L - 1 && h->drec && has_dprev && !dropout_prev && !recorder(h)) {
                // implicit delta_{L-1}: gather the records the output layer's backward just wrote
                A.drec = h->drec;
                A.dL = h->delta[L] + (int64_t)c * h->sizes[L - 1] * CB;
                A.rc_slope = neg_slope_of(h, l);
                A.zero_row = (int)nout;
            }
            // (implicit delta_l: 16-B records instead of the delta_l rows)
            const double dl_bytes = A.drec ? 4.0 * Bc * (double)nout - 16.0 * (double)nout : 0.0;
            prof_start(h, K_BWD, l, 12.0 * nnz / nchunks + act_bytes - dl_bytes, (has_dprev ? 4.0 : 2.0) * nnz * Bc);
            SMLP_TRY(dispatch_bwd(h, A, Ly, has_dprev));
            prof_stop(h);
            if (last) SMLP_TRY(layer_done(h, l));
        }
    }
    if (early && h->xbits && !recorder(h) && h->param_count > SMALL_MODEL_PARAMS) {
        // fused step of a large model with the bit path: the gradients of W^(3..L) are final, and what
        // is left of the backward (the set-bit walk of W^(2), bound by latency and instruction issue)
        // leaves the memory system idle -- so Eq. 1 and the mirror refresh of those layers (streaming
        // and gather passes) run on the side stream under it; run_step joins them
        SMLP_TRY(ensure_aux(h));
        SMLP_CK(h, cudaEventRecord(h->aux_ev[0], h->stream));
        SMLP_CK(h, cudaStreamWaitEvent(h->aux_stream, h->aux_ev[0], 0));
        for (auto& Ly : h->layers) {
            if (Ly.l < 3) continue;
            const bool g2 = Ly.split;
            Ly.split = false;
            SMLP_TRY(launch_update(h, h->aux_stream, Ly.val_off, Ly.val_off + Ly.cap, true, early, g2));
            Ly.updated_early = true;
            if (Ly.narrow) continue;
            mirror_values_kernel<<<launch_grid(h, (Ly.cap + 3) / 4, 256), 256, 0, h->aux_stream>>>(Ly.val, Ly.mperm, Ly.meta,
                                                                                         Ly.mval);
            SMLP_CK_LAUNCH(h, "mirror_values_kernel");
        }
    }
    if (h->xbits) {   // binary-input layer 2 (returns at once if not binary)
        Layer& L2 = h->layers[0];
        BitsArgs A = bits_args(h, L2, nchunks);
        const double nnz = (double)L2.nnz;
        prof_start(h, K_BWD_BITS, 2, 8.0 * nnz + 4.0 * B * (double)(L2.n_in + L2.n_out), 2.0 * nnz * B);   // src, g
        SMLP_TRY(dispatch_bits(h, A, L2, false));
        prof_stop(h);
        prof_start(h, K_LAYER_UPDATE, 2, 12.0 * nnz, 0.0);
        const MirrorGradArgs MG{h->d_nonbinary, h->gmirror2, L2.minv, L2.grad, L2.meta};
        if (Recorder* R = recorder(h)) {
            if (PPhase* ph = R->add(PK_GRAD_FROM_MIRROR, 0, 0, 0)) ph->a.mg = MG;
        } else {
            launch_pdl(h->pdl, grad_from_mirror_kernel, launch_grid(h, L2.cap, 256), 256, h->stream, MG);
            SMLP_CK_LAUNCH(h, "grad_from_mirror_kernel");
        }
        prof_stop(h);
        SMLP_TRY(layer_done(h, 2));
    }
    return SMLP_OK;
}

int run_step(smlp_handle* h, const smlp_sgd* sgd) {
    // Eq. 1 per layer slice on the handle's stream; each layer's mirror refresh (a gather, bound by
    // L2 requests rather than HBM bytes) runs on a side stream as soon as that slice is updated, so
    // it overlaps the next slice's streaming update
    const int64_t n = h->param_count;
    if (n <= SMALL_MODEL_PARAMS) {
        // small models are launch-bound: one Eq. 1 launch over the whole view (decay below
        // bias_base) and one mirror refresh for all layers, both on the handle's stream
        prof_start(h, K_SGD, 0, 20.0 * (double)n, 0.0);
        SMLP_TRY(launch_update(h, h->stream, 0, n, true, sgd));
        MirrorSet M{};
        int nl = 0;
        int64_t cmax = 1;
        for (auto& Ly : h->layers) {
            if (Ly.narrow) continue;                               // narrow layers never read the mirror copy
            M.val[nl] = Ly.val;
            M.mperm[nl] = Ly.mperm;
            M.meta[nl] = Ly.meta;
            M.mval[nl] = Ly.mval;
            cmax = std::max<int64_t>(cmax, Ly.cap);
            ++nl;
        }
        if (nl > 0) {
            const dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>((cmax + 255) / 256, h->num_sms * 4)),
                            (unsigned)nl);
            if (Recorder* R = recorder(h)) {
                R->P.mirror = M;
                R->add(PK_MIRROR, (int)grid.x, (int)grid.y, 0);
            } else {
                launch_pdl(h->pdl, mirror_values_multi_kernel, grid, 256, h->stream, M);
                SMLP_CK_LAUNCH(h, "mirror_values_multi_kernel");
            }
        }
        prof_stop(h);
        return SMLP_OK;
    }
    if (Recorder* R = recorder(h)) {   // large models: per-layer slices + side-stream refreshes
        R->ok = false;
        return SMLP_OK;
    }
    SMLP_TRY(ensure_aux(h));
    auto update = [&](int64_t lo, int64_t hi, bool decay) { return launch_update(h, h->stream, lo, hi, decay, sgd); };
    prof_start(h, K_SGD, 0, 20.0 * (double)n, 0.0);
    bool side = false;
    for (auto& Ly : h->layers) {
        if (Ly.updated_early) {   // issued on the side stream by the backward (under the bit kernels)
            Ly.updated_early = false;
            side = true;
            continue;
        }
        const bool g2 = Ly.split;
        Ly.split = false;
        SMLP_TRY(launch_update(h, h->stream, Ly.val_off, Ly.val_off + Ly.cap, true, sgd, g2));
        if (Ly.narrow) continue;                                   // narrow layers never read the mirror copy
        SMLP_CK(h, cudaEventRecord(h->aux_ev[0], h->stream));
        SMLP_CK(h, cudaStreamWaitEvent(h->aux_stream, h->aux_ev[0], 0));
        mirror_values_kernel<<<launch_grid(h, (Ly.cap + 3) / 4, 256), 256, 0, h->aux_stream>>>(Ly.val, Ly.mperm, Ly.meta,
                                                                                     Ly.mval);
        SMLP_CK_LAUNCH(h, "mirror_values_kernel");
        side = true;
    }
    SMLP_TRY(update(h->bias_base, n, false));                      // biases: no weight decay
    if (side) {
        SMLP_CK(h, cudaEventRecord(h->aux_ev[1], h->aux_stream));
        SMLP_CK(h, cudaStreamWaitEvent(h->stream, h->aux_ev[1], 0));
    }
    prof_stop(h);
    return SMLP_OK;
}

// ------------------------------------------------------------------------------------------
// persistent step: launch of a recorded program (one cooperative wave), and the API-level entry
// points that record when the handle takes the persistent path (h->persist) and fall back to
// the per-kernel launches when a call needs a phase the persistent kernel does not carry
// ------------------------------------------------------------------------------------------
static_assert(sizeof(PProgram) <= 32000, "the phase list is passed as one kernel parameter");

template <int CB>
static int launch_persist_cb(smlp_handle* h, const PProgram& P) {
    static int per_sm = 0;
    const size_t smem = sizeof(PersistSmem<CB>);
    if (per_sm == 0) {
        SMLP_CK(h, cudaFuncSetAttribute(persist_step_kernel<CB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        SMLP_CK(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, persist_step_kernel<CB>, 256, smem));
        if (per_sm < 1) return set_err(h, SMLP_E_CUDA, "persistent step kernel does not fit an SM");
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(per_sm * h->num_sms));
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = h->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    SMLP_CK(h, cudaLaunchKernelEx(&cfg, persist_step_kernel<CB>, P));
    SMLP_CK_LAUNCH(h, "persist_step_kernel");
#ifdef SMLP_PERSIST_TIMING
    {
        unsigned long long t[PMAX + 1];
        cudaStreamSynchronize(h->stream);
        cudaMemcpyFromSymbol(t, g_phase_ns, sizeof(t));
        unsigned long long prev = t[PMAX];
        fprintf(stderr, "persist phases:");
        for (int i = 0; i < P.n; ++i) {
            fprintf(stderr, " %d:%.1f", P.ph[i].kind, (double)(t[i] - prev) / 1e3);
            prev = t[i];
        }
        fprintf(stderr, " us\n");
    }
#endif
    return SMLP_OK;
}

static int launch_persist(smlp_handle* h, PProgram& P, int prof_kind, double bytes, double flops) {
    P.bar = h->gbar;
    P.smslot = h->gbar + 2;
    P.nsm = h->num_sms;
    prof_start(h, prof_kind, 0, bytes, flops);
    int rc;
    switch (h->CB) {
        case 8: rc = launch_persist_cb<8>(h, P); break;
        case 16: rc = launch_persist_cb<16>(h, P); break;
        case 32: rc = launch_persist_cb<32>(h, P); break;
        case 64: rc = launch_persist_cb<64>(h, P); break;
        case 128: rc = launch_persist_cb<128>(h, P); break;
        default: rc = set_err(h, SMLP_E_ARG, "persistent step: unsupported chunk_batch");
    }
    prof_stop(h);
    return rc;
}

// Records the phases `body` would launch; returns 1 (and leaves nothing enqueued) when the call
// must take the per-kernel path instead.
template <typename F>
static int record_program(smlp_handle* h, Recorder& R, F&& body, int* rc) {
    R.P.n = 0;
    R.ok = true;
    h->rec = &R;
    h->rec_bytes = h->rec_flops = 0.0;
    *rc = body();
    h->rec = nullptr;
    return (*rc == SMLP_OK && R.ok && R.P.n > 0) ? 0 : 1;
}

int run_forward(smlp_handle* h, const float* x, const int32_t* x_idx, int B, bool train, uint64_t step,
                float* probs) {
    if (h->persist) {
        Recorder R;
        int rc;
        if (record_program(h, R, [&] { return run_forward_phases(h, x, x_idx, B, train, step, probs); }, &rc) == 0)
            return launch_persist(h, R.P, K_PERSIST_FWD, h->rec_bytes, h->rec_flops);
        if (rc != SMLP_OK) return rc;
    }
    return run_forward_phases(h, x, x_idx, B, train, step, probs);
}

// backward (a4-a5) and, when fused, the Eq. 1 pass + mirror refresh (a6) of the same call
int run_backward_step(smlp_handle* h, const int32_t* labels, const int32_t* y_idx, float* loss, const smlp_sgd* fused) {
    auto body = [&]() -> int {
        SMLP_TRY(run_backward_phases(h, labels, y_idx, loss, fused != nullptr, fused));
        if (fused) SMLP_TRY(run_step(h, fused));
        return SMLP_OK;
    };
    if (h->persist) {
        Recorder R;
        int rc;
        if (record_program(h, R, body, &rc) == 0) {
            SMLP_TRY(launch_persist(h, R.P, K_PERSIST_BWD, h->rec_bytes, h->rec_flops));
            for (int l = h->L; l >= 2; --l) SMLP_TRY(layer_done(h, l));   // every layer final at once
            return SMLP_OK;
        }
        if (rc != SMLP_OK) return rc;
    }
    return body();
}

int run_backward(smlp_handle* h, const int32_t* labels, const int32_t* y_idx, float* loss, bool split_last) {
    return run_backward_phases(h, labels, y_idx, loss, split_last);
}

}  // namespace smlp
