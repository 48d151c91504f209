// smlp_internal.cuh — internal state and device helpers of libsparse_mlp.so (sm_100a).
//
// Layout in HBM:
//   param / mom / grad : one contiguous fp32 buffer each, [W^(2) cap | ... | W^(L) cap | b_2 | ... | b_L]
//                        (offsets rounded to 32 floats) — the grad view is what a multi-GPU
//                        step allreduces (X1), the param view what averaging allreduces (X2).
//   W^(l) canonical    : input-major CSR (the paper orientation): row_ptr int32
//                        [n_{l-1}+1], col int32 [cap], val/mom/grad fp32 slices [cap], rowid int32
//                        [cap] (row of each entry, for nnz-parallel kernels).
//   W^(l) mirror       : output-major CSR: mrow_ptr [n_l+1], msrc [cap] (input neuron i),
//                        mperm [cap] (canonical index of the entry).
//   activations        : "chunked transposed": act[l] = [n_chunks][n_l][CB] fp32, CB = chunk_batch
//                        batch columns per chunk, so one neuron's CB values are one contiguous
//                        row (CB = 128 -> 512 B, one float4 per lane of a warp).  The forward
//                        tensors (act, zmask, kmask) use their own width CBf <= CB (CB / CBf
//                        forward chunks per backward chunk); delta uses CB.
//   masks              : per hidden neuron row and chunk, uint4 = 4 x 32 bits; word c, bit q
//                        is batch column 4q + c of the chunk (one ballot per float4 lane).
//   work lists         : per layer, forward segments over mirror rows and backward segments
//                        over canonical rows, each <= SEG_NNZ entries, counts in device memory.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/sparse_mlp.h"

namespace smlp {

constexpr int SEG_NNZ = 64;               // max nnz per work segment (long-row split; one row-kernel window)
constexpr int WARPS_PER_BLOCK = 8;        // 256-thread blocks for the warp-per-row kernels
constexpr int NARROW_MAX = 32;            // output layers with n_L <= 32 take the narrow path
constexpr int NARROW_MAX_ELEMS = 2048;    // ... if next_pow2(n_L) x chunk_batch <= this
constexpr int NARROW_WARPS = 8;
constexpr int64_t SMALL_MODEL_PARAMS = 1 << 22;   // run_step: one update + one mirror launch at or below this
constexpr int XBITS_WORDS = 4;          // bit-packed input: 128 batch columns per input neuron

struct LayerMeta {                         // device-resident counts (graph-stable)
    int32_t nnz;
    int32_t n_fseg;
    int32_t n_bseg;
    int32_t n_fmulti;
    int32_t n_bmulti;
    int32_t pad[3];
};

struct Layer {
    int l = 0;
    int64_t n_in = 0, n_out = 0;
    bool dense = false;
    int64_t cap = 0, nnz = 0;
    int64_t val_off = 0, bias_off = 0;
    // canonical CSR
    int32_t* row_ptr = nullptr;
    int32_t* col = nullptr;
    int32_t* rowid = nullptr;
    float* val = nullptr;
    float* mom = nullptr;
    float* grad = nullptr;
    // output-major mirror
    int32_t* mrow_ptr = nullptr;
    int32_t* msrc = nullptr;
    int32_t* mperm = nullptr;
    int32_t* minv = nullptr;    // canonical index -> mirror position (inverse of mperm)
    float* mval = nullptr;      // mirror-ordered copy of val (the forward reads it sequentially)
    // segment work lists: int4 (row, beg, end, slot) ; multi: int4 (row, first_slot, n_slots, 0)
    int64_t fseg_cap = 0, bseg_cap = 0, fslot_cap = 0, bslot_cap = 0;
    int4* fseg = nullptr;
    int4* bseg = nullptr;
    int4* fmulti = nullptr;
    int4* bmulti = nullptr;
    float* fws = nullptr;   // [fslot_cap][CB] partial sums of multi-segment forward rows
    float* bws = nullptr;   // [bslot_cap][CB] partial delta sums of multi-segment backward rows
    float* bgs = nullptr;   // [n_in] bias-grad accumulator across chunks (for layer l-1)
    LayerMeta* meta = nullptr;
    LayerMeta meta_h{};
    // narrow output layer path (l = L, n_L <= NARROW_MAX): canonical-row streaming fwd / bwd
    bool narrow = false;
    int nout_pad = 0;       // next power of two >= n_out (>= 2)
    int ngrid = 0;          // CTAs of the narrow forward
    float* nws = nullptr;   // [ngrid][nout_pad][CB] CTA partial logits
    bool split = false;     // the last backward chunk's gradient is in grad2 (the Eq. 1 pass adds it)
    bool updated_early = false;  // Eq. 1 + mirror refresh already issued on the side stream by this backward (run_step skips it)
    bool narrow_bwd = false; // the backward of a narrow layer streams its rows too (dense-capped only by default)
    // biases of neuron layer l live in param/mom/grad at bias_off
    float* bias = nullptr;
    float* bias_mom = nullptr;
    float* bias_grad = nullptr;
};

struct Alloc {
    size_t bytes;
    void* ptr;
};

enum KernelKind { K_STAGE = 0, K_FWD = 1, K_FWD_FINISH = 2, K_SOFTMAX = 3, K_BWD = 4, K_BWD_FINISH = 5, K_SGD = 6,
                  K_FWD_BITS = 7, K_BWD_BITS = 8, K_LAYER_UPDATE = 9, K_MIRROR = 10, K_PERSIST_FWD = 11,
                  K_PERSIST_BWD = 12 };

struct ProfRec {
    int kind, layer;
    cudaEvent_t a, b;
    double bytes, flops;
};

}  // namespace smlp

struct smlp_handle {
    int L = 0;
    int64_t sizes[SMLP_MAX_LAYERS] = {0};
    double eps = 0;
    int activation = SMLP_ACT_ALL_RELU;
    float alpha = 0.f, dropout = 0.f;
    int init = SMLP_INIT_HE_U;
    uint64_t seed = 0;
    int rank = 0;
    int max_batch = 0;
    int CB = 128;           // backward chunk width (delta layout)
    int max_chunks = 1;
    int CBf = 128;          // forward chunk width (act / zmask / kmask layout), CB % CBf == 0
    int max_chunks_f = 1;
    int device = 0;
    cudaStream_t stream = nullptr;
    smlp_allocator allocator{};
    bool has_allocator = false;
    std::vector<smlp::Alloc> allocs;   // every live allocation (freed at destroy)

    std::vector<smlp::Layer> layers;   // layers[l-2] = W^(l)
    float* param = nullptr;
    float* mom = nullptr;
    float* grad = nullptr;
    float* grad2 = nullptr;         // large models: the last chunk's gradient of the fused path
    int64_t param_count = 0;
    int64_t bias_base = 0;

    float* act[SMLP_MAX_LAYERS + 1] = {nullptr};     // index l (1..L)
    float* delta[SMLP_MAX_LAYERS + 1] = {nullptr};   // index l (2..L)
    uint4* zmask[SMLP_MAX_LAYERS + 1] = {nullptr};   // hidden l: bit = (z > 0)
    uint4* kmask[SMLP_MAX_LAYERS + 1] = {nullptr};   // hidden l: bit = dropout keep
    uint8_t* alive[SMLP_MAX_LAYERS + 1] = {nullptr}; // index l (1..L)
    int64_t alive_h[SMLP_MAX_LAYERS + 1] = {0};

    int32_t* d_err = nullptr;       // label-range flag
    uint32_t* xbits = nullptr;      // [n_1][XBITS_WORDS] bit-packed input (binary-input path) or null
    int32_t* d_nonbinary = nullptr; // set by stage_input when an input value is not 0 or 1
    float* gmirror2 = nullptr;      // [cap of W^(2)] gradient in mirror order (binary-input path)
    // implicit delta_{L-1}: per neuron j of layer L-1 and backward chunk, the sign bits of
    // z_{L-1}[j] over the chunk's columns and the two weights of row j of a dense-capped 2-output
    // W^(L) -- written by the output layer's backward, gathered (16 B instead of a 4 CB-byte
    // delta row) by the backward of W^(L-1), which recomputes delta_{L-1}[j] from it and delta_L
    uint4* drec = nullptr;          // [n_{L-1} + 1], the last record all zero (padding slots)
    bool implicit_delta = true;
    float* d_loss = nullptr;        // scratch loss for train_step_host
    float* x_stage[2] = {nullptr, nullptr};   // [max_batch x n_1] x2 for train_step_host (double-buffered)
    int32_t* y_stage[2] = {nullptr, nullptr};
    cudaStream_t copy_stream = nullptr;        // H2D of the next host batch, overlapping the current step
    cudaStream_t aux_stream = nullptr;         // mirror refreshes overlapping the Eq. 1 pass (run_step)
    cudaEvent_t aux_ev[2] = {nullptr, nullptr};
    cudaEvent_t ev_copied[2] = {nullptr, nullptr};
    cudaEvent_t ev_consumed[2] = {nullptr, nullptr};
    int stage_idx = 0;
    cudaEvent_t layer_ev[SMLP_MAX_LAYERS + 1] = {nullptr};   // W^(l) gradient final (unfused backward)

    // trace of the last forward
    bool trace_valid = false;
    bool trace_train = false;
    int trace_B = 0;
    uint64_t trace_version = 0;
    uint64_t trace_step = 0;
    bool grads_pending = false;

    uint64_t version = 0;
    const uint64_t* step_counter = nullptr;   // device dropout-step source (graph replay)
    bool prof = false;
    std::vector<smlp::ProfRec> prof_recs;
    std::vector<cudaEvent_t> ev_pool;
    int num_sms = 148;
    int pdl = 0;                    // launch the step's kernels with programmatic serialization
    int persist = 0;                // small models: every forward / backward call is one persistent launch
    void* rec = nullptr;            // persistent step: the phase recorder while a call records (step.cu)
    unsigned* gbar = nullptr;       // persistent step: grid barrier [count, generation], then per-SM slot counters
    double rec_bytes = 0.0, rec_flops = 0.0;   // ... and the algorithmic bytes / flops of its phases
    // tuning knobs (env, read at create; each selects between kernels the parity tests cover)
    int narrow_sparse_bwd = 0;      // SMLP_NARROW_SPARSE_BWD: narrow row-streaming backward also for a sparse output layer
    int64_t short_min_rows = -1;    // SMLP_SHORT_MIN_ROWS: -1 = one 32-row unit per resident warp
    int short_max_fwd = 16;         // SMLP_SHORT_MAX_FWD / _BWD: average entries per row below which the
    int short_max_bwd = 8;          //   streaming kernels run (T2/T3 at ~10: forward -5%, backward +80%)
    bool input_binary = false;      // SMLP_INPUT_BINARY: inputs promised {0,1}; a broken promise is reported
    int64_t launches = 0;
    std::string err;
};

namespace smlp {

// ------------------------------------------------------------------------------------------
// error helpers
// ------------------------------------------------------------------------------------------
int set_err(smlp_handle* h, int code, const std::string& msg);
int check_cuda(smlp_handle* h, cudaError_t e, const char* what);
#define SMLP_CK(h, call)                                                   \
    do {                                                                   \
        cudaError_t _e = (call);                                           \
        if (_e != cudaSuccess) return ::smlp::check_cuda((h), _e, #call);  \
    } while (0)
#define SMLP_CK_LAUNCH(h, what)                                            \
    do {                                                                   \
        (h)->launches++;                                                   \
        cudaError_t _e = cudaGetLastError();                               \
        if (_e != cudaSuccess) return ::smlp::check_cuda((h), _e, what);   \
    } while (0)
#define SMLP_TRY(call)             \
    do {                           \
        int _rc = (call);          \
        if (_rc != SMLP_OK) return _rc; \
    } while (0)

// ------------------------------------------------------------------------------------------
// Programmatic dependent launch ("launch chain"): for small models (h->pdl) the
// step's kernels are launched with the programmatic-serialization attribute, so kernel n+1's
// launch and CTA rasterisation overlap kernel n's tail; every such kernel starts with
// SMLP_PDL_ENTRY -- griddepcontrol.wait blocks until the previous grid has COMPLETED and its
// writes are visible (so no kernel reads a predecessor's output early), then launch_dependents
// lets the next grid start launching.  Without the attribute both are no-ops.
// ------------------------------------------------------------------------------------------
#define SMLP_PDL_ENTRY()                                          \
    do {                                                          \
        asm volatile("griddepcontrol.wait;" ::: "memory");        \
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); \
    } while (0)

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(int pdl, void (*kernel)(KArgs...), dim3 grid, dim3 block, cudaStream_t stream,
                              Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = 0;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, args...);
}

// Device bounds checks ("bounds-checked build"): compiled in only by the A/B build
// tools/ab_build.py bounds -DSMLP_BOUNDS_CHECK=1 (compute-sanitizer is closed on the GPU pool), which
// the GPU parity tests then run against with SMLP_LIB; a violated bound prints and traps.
#ifdef SMLP_BOUNDS_CHECK
#define SMLP_BOUND(cond, what)                                                             \
    do {                                                                                   \
        if (!(cond)) {                                                                     \
            printf("smlp bounds check failed: %s (%s:%d)\n", what, __FILE__, __LINE__);   \
            __trap();                                                                      \
        }                                                                                  \
    } while (0)
#else
#define SMLP_BOUND(cond, what) \
    do {                       \
    } while (0)
#endif

// per-kernel CUDA-event timing (no-ops unless h->prof)
void prof_start(smlp_handle* h, int kind, int layer, double bytes, double flops);
void prof_stop(smlp_handle* h);

// allocation through the caller's allocator (or cudaMallocAsync); tracked for destroy
void* dev_alloc(smlp_handle* h, size_t bytes);
void dev_free(smlp_handle* h, void* p);
// temporary allocation freed by the caller with tmp_free (not tracked)
void* tmp_alloc(smlp_handle* h, size_t bytes);
void tmp_free(smlp_handle* h, void* p, size_t bytes);

// ------------------------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al., SC'11) and the stream layout of DESIGN.md (R2, R8, R13)
// ------------------------------------------------------------------------------------------
enum Purpose : uint32_t { P_INIT = 1, P_INIT_DENSE = 2, P_REGROW = 3, P_DROPOUT = 4 };

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
        if (r < 9) {
            k.x += 0x9E3779B9u;
            k.y += 0xBB67AE85u;
        }
    }
    return c;
}

__device__ __forceinline__ uint4 rng_stream(uint64_t seed, uint32_t purpose, uint32_t rank,
                                            uint32_t layer, uint32_t c3, uint64_t idx) {
    const uint4 c = make_uint4((uint32_t)idx, (uint32_t)(idx >> 32),
                               ((purpose & 0xffu) << 24) | ((rank & 0xffu) << 16) | (layer & 0xffffu), c3);
    return philox4x32_10(c, make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
}

// candidate position from two uniform words: i = floor(x0 n_in / 2^32), j likewise
__device__ __forceinline__ uint32_t scale_u32(uint32_t x, uint64_t n) {
    return (uint32_t)(((uint64_t)x * n) >> 32);
}

// Initial / regrown value (R3, R4): uniform schemes are exact but for the final fp32 multiply;
// "normal" is Box-Muller in fp64 rounded once to fp32.
struct InitParams {
    int scheme;
    float lim;      // fp32(sqrt(6/n_in)) or fp32(sqrt(6/(n_in+n_out)))
    double std;     // sqrt(2/n_in)
};

__device__ __forceinline__ float init_value(const InitParams& p, uint32_t x2, uint32_t x3) {
    if (p.scheme != SMLP_INIT_NORMAL) {
        const float u = __fmul_rn((float)(x2 >> 8), 5.9604644775390625e-08f);
        const float t = __fadd_rn(__fmul_rn(u, 2.0f), -1.0f);
        return __fmul_rn(t, p.lim);
    }
    const double u1 = __dmul_rn((double)(x2 >> 8) + 1.0, 5.9604644775390625e-08);
    const double u2 = __dmul_rn((double)(x3 >> 8), 5.9604644775390625e-08);
    const double r = sqrt(__dmul_rn(-2.0, log(u1)));
    const double c = cos(__dmul_rn(6.283185307179586, u2));
    return (float)__dmul_rn(__dmul_rn(r, c), p.std);
}

InitParams init_params(const smlp_handle* h, const Layer& L);

// ------------------------------------------------------------------------------------------
// topology build helpers (topology.cu)
// ------------------------------------------------------------------------------------------
// From a canonical CSR (row_ptr, col filled for nnz entries) rebuild rowid, the output-major
// mirror and both segment work lists; refreshes meta (device + host).
int rebuild_derived(smlp_handle* h, Layer& L);
// Sorted unique positions (u64 pos = i * n_out + j) with values -> canonical CSR arrays of L
// (row_ptr, col, val; mom zeroed) for n entries.  pos/val are device arrays.
int csr_from_sorted_positions(smlp_handle* h, Layer& L, const uint64_t* pos, const float* val,
                              int64_t n);
// "First R distinct valid candidates in stream order" (R2, R8): candidates m = 0.. of stream
// (purpose, layer, c3); valid = not in the current support of L (if exclude_support) and both
// neurons alive (if alive_in/alive_out non-NULL).  Output: R positions sorted ascending and
// their values (init scheme).  out_pos/out_val are device arrays of >= R elements.
int first_distinct_candidates(smlp_handle* h, const Layer& L, uint32_t purpose, uint32_t c3,
                              int64_t R, bool exclude_support, const uint8_t* alive_in,
                              const uint8_t* alive_out, int64_t n_free, uint64_t* out_pos,
                              float* out_val);
int fill_dense_layer(smlp_handle* h, Layer& L);
// zero val / mom / grad (and the fused path's grad2) of W^(l) beyond its first n entries, so the
// param / grad views hold zeros in [nnz, cap) and the Eq. 1 pass leaves that tail at zero
int zero_tail(smlp_handle* h, Layer& L, int64_t n);
int launch_grid(const smlp_handle* h, int64_t items, int threads);

// step.cu
int run_forward(smlp_handle* h, const float* x, const int32_t* x_idx, int B, bool train,
                uint64_t step, float* probs);
// the gradient of the current trace into the grad view (split_last: a large model's last chunk
// into grad2, added by the Eq. 1 pass that follows in the same call)
int run_backward(smlp_handle* h, const int32_t* labels, const int32_t* y_idx, float* loss, bool split_last);
// backward (+ the fused Eq. 1 pass when fused != null); one persistent launch for small models
int run_backward_step(smlp_handle* h, const int32_t* labels, const int32_t* y_idx, float* loss, const smlp_sgd* fused);
int run_step(smlp_handle* h, const smlp_sgd* sgd);
int refresh_mirror_values(smlp_handle* h, Layer& Ly);

// evolve.cu / prune.cu
int run_evolve(smlp_handle* h, double zeta, uint64_t e, int64_t* removed);
int run_importance(smlp_handle* h, int l, double* out_dev);
int run_prune(smlp_handle* h, double rho, int flags, int64_t* pruned, int64_t* removed);
// compact W^(l) to the entries whose flag is 0 (no additions), rebuild derived state
int compact_layer(smlp_handle* h, Layer& L, const uint8_t* remove_flags);
// merge: survivors (flag 0) of L plus R sorted additions (pos, val) -> new canonical CSR
int merge_layer(smlp_handle* h, Layer& L, const uint8_t* remove_flags, const uint64_t* add_pos,
                const float* add_val, int64_t R);

}  // namespace smlp
