// api.cu — the extern "C" boundary of libsparse_mlp.so (include/sparse_mlp.h).
//
// Host-side bookkeeping only: argument validation, allocation, trace / version state, and the
// small synchronous copies of the parity / checkpoint paths.  Every step of the method runs in
// the kernels of step.cu, topology.cu, evolve.cu and prune.cu; there is no CPU fallback.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "smlp_internal.cuh"

namespace {
thread_local std::string g_create_error;
}

namespace smlp {

int set_err(smlp_handle* h, int code, const std::string& msg) {
    if (h) h->err = msg; else g_create_error = msg;
    return code;
}

int check_cuda(smlp_handle* h, cudaError_t e, const char* what) {
    return set_err(h, SMLP_E_CUDA, std::string("CUDA error ") + cudaGetErrorString(e) + " in " + what);
}

void* tmp_alloc(smlp_handle* h, size_t bytes) {
    bytes = std::max<size_t>(bytes, 16);
    void* p = nullptr;
    if (h->has_allocator) {
        p = h->allocator.alloc(bytes, (void*)h->stream, h->allocator.ctx);
    } else if (cudaMallocAsync(&p, bytes, h->stream) != cudaSuccess) {
        p = nullptr;
    }
    return p;
}

void tmp_free(smlp_handle* h, void* p, size_t bytes) {
    if (!p) return;
    bytes = std::max<size_t>(bytes, 16);
    if (h->has_allocator) h->allocator.free(p, bytes, (void*)h->stream, h->allocator.ctx);
    else cudaFreeAsync(p, h->stream);
}

void* dev_alloc(smlp_handle* h, size_t bytes) {
    void* p = tmp_alloc(h, bytes);
    if (p) h->allocs.push_back({std::max<size_t>(bytes, 16), p});
    return p;
}

void dev_free(smlp_handle* h, void* p) {
    for (size_t k = 0; k < h->allocs.size(); ++k) {
        if (h->allocs[k].ptr == p) {
            tmp_free(h, p, h->allocs[k].bytes);
            h->allocs.erase(h->allocs.begin() + (long)k);
            return;
        }
    }
}

// inside a CUDA-graph capture the profiling events become external event-record nodes, so every
// replay re-stamps them and the kernel times of the last replay can be read back
static void prof_record(smlp_handle* h, cudaEvent_t e) {
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(h->stream, &st) == cudaSuccess && st == cudaStreamCaptureStatusActive)
        cudaEventRecordWithFlags(e, h->stream, cudaEventRecordExternal);
    else
        cudaEventRecord(e, h->stream);
}

void prof_start(smlp_handle* h, int kind, int layer, double bytes, double flops) {
    if (h->rec) {            // recording a persistent step: its launch is timed as one record
        h->rec_bytes += bytes;
        h->rec_flops += flops;
        return;
    }
    if (!h->prof) return;
    ProfRec r{kind, layer, nullptr, nullptr, bytes, flops};
    for (cudaEvent_t* e : {&r.a, &r.b}) {
        if (!h->ev_pool.empty()) {
            *e = h->ev_pool.back();
            h->ev_pool.pop_back();
        } else {
            cudaEventCreate(e);
        }
    }
    prof_record(h, r.a);
    h->prof_recs.push_back(r);
}

void prof_stop(smlp_handle* h) {
    if (h->rec || !h->prof || h->prof_recs.empty()) return;
    prof_record(h, h->prof_recs.back().b);
}

}  // namespace smlp

using namespace smlp;

namespace {

template <typename T>
T* zalloc(smlp_handle* h, size_t count, int* rc) {
    if (*rc != SMLP_OK) return nullptr;
    T* p = (T*)dev_alloc(h, sizeof(T) * std::max<size_t>(count, 1));
    if (!p) {
        *rc = set_err(h, SMLP_E_NOMEM, "device allocation failed");
        return nullptr;
    }
    if (cudaMemsetAsync(p, 0, sizeof(T) * std::max<size_t>(count, 1), h->stream) != cudaSuccess) {
        *rc = set_err(h, SMLP_E_CUDA, "cudaMemsetAsync failed");
    }
    return p;
}

int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

int next_pow2(int v) {
    int p = 1;
    while (p < v) p <<= 1;
    return p;
}

bool valid_layer(const smlp_handle* h, int l, int lo) { return h && l >= lo && l <= h->L; }

int check_data_flag(smlp_handle* h) {
    int32_t flag = 0;
    if (cudaMemcpyAsync(&flag, h->d_err, 4, cudaMemcpyDeviceToHost, h->stream) != cudaSuccess)
        return set_err(h, SMLP_E_CUDA, "error-flag read");
    if (cudaStreamSynchronize(h->stream) != cudaSuccess) return set_err(h, SMLP_E_CUDA, "sync");
    if (flag) {
        cudaMemsetAsync(h->d_err, 0, 4, h->stream);
        if (flag & 2) return set_err(h, SMLP_E_DATA, "an input value outside {0, 1} with SMLP_INPUT_BINARY");
        return set_err(h, SMLP_E_DATA, "a label outside [0, n_L) was passed to backward");
    }
    return SMLP_OK;
}

int build_handle(smlp_handle* h, const smlp_config* cfg) {
    int rc = SMLP_OK;
    const int L = h->L;
    // --- layer shapes, capacities and param layout
    h->layers.resize((size_t)(L - 1));
    int64_t off = 0;
    for (int l = 2; l <= L; ++l) {
        Layer& Ly = h->layers[(size_t)(l - 2)];
        Ly.l = l;
        Ly.n_in = h->sizes[l - 2];
        Ly.n_out = h->sizes[l - 1];
        const double total = (double)Ly.n_in * (double)Ly.n_out;
        const double m = std::floor(h->eps * (double)(Ly.n_in + Ly.n_out));
        const double M = std::min(total, m);
        if (M >= 2147483647.0) return set_err(h, SMLP_E_ARG, "layer " + std::to_string(l) + ": nnz >= 2^31");
        Ly.cap = (int64_t)M;
        Ly.dense = (M == total);
        Ly.val_off = off;
        off += round_up(std::max<int64_t>(Ly.cap, 1), 32);
    }
    h->bias_base = off;
    for (int l = 2; l <= L; ++l) {
        Layer& Ly = h->layers[(size_t)(l - 2)];
        Ly.bias_off = off;
        off += round_up(Ly.n_out, 32);
    }
    h->param_count = off;
    // programmatic dependent launch for the launch-bound small models only (measured
    // C4 / C3 -2..5%, C5 +12% per step)
    h->pdl = off <= SMALL_MODEL_PARAMS ? 1 : 0;
    h->gbar = zalloc<unsigned>(h, 2 + (size_t)h->num_sms, &rc);   // barrier [count, gen] + per-SM slot counters
    // persistent step: built and bit-identical to the per-kernel path, but measured
    // 1.4-1.9x slower than the CUDA-graph replay of the per-kernel step on C1-C4, so it is opt-in:
    // SMLP_PERSIST=1 (small models whose forward and backward tensors share one chunk width)
    h->persist = 0;
    if (const char* e = std::getenv("SMLP_PERSIST"))
        h->persist = (std::atoi(e) != 0 && off <= SMALL_MODEL_PARAMS && h->CB == h->CBf && h->CB >= 8) ? 1 : 0;
    h->param = zalloc<float>(h, (size_t)off, &rc);
    h->mom = zalloc<float>(h, (size_t)off, &rc);
    h->grad = zalloc<float>(h, (size_t)off, &rc);
    // the fused path's last backward chunk writes its own gradient buffer, so no chunk kernel
    // re-reads the earlier chunks' sum (the Eq. 1 pass adds the two); large models only
    if (off > SMALL_MODEL_PARAMS) h->grad2 = zalloc<float>(h, (size_t)off, &rc);
    if (rc) return rc;
    const int CB = h->CB;
    for (auto& Ly : h->layers) {
        Ly.val = h->param + Ly.val_off;
        Ly.mom = h->mom + Ly.val_off;
        Ly.grad = h->grad + Ly.val_off;
        Ly.bias = h->param + Ly.bias_off;
        Ly.bias_mom = h->mom + Ly.bias_off;
        Ly.bias_grad = h->grad + Ly.bias_off;
        const size_t cap = (size_t)std::max<int64_t>(Ly.cap, 1);
        Ly.row_ptr = zalloc<int32_t>(h, (size_t)Ly.n_in + 1, &rc);
        Ly.col = zalloc<int32_t>(h, cap, &rc);
        Ly.rowid = zalloc<int32_t>(h, cap, &rc);
        Ly.mrow_ptr = zalloc<int32_t>(h, (size_t)Ly.n_out + 1, &rc);
        Ly.msrc = zalloc<int32_t>(h, cap, &rc);
        Ly.mperm = zalloc<int32_t>(h, cap, &rc);
        Ly.minv = zalloc<int32_t>(h, cap, &rc);
        Ly.mval = zalloc<float>(h, cap, &rc);
        Ly.fseg_cap = Ly.n_out + Ly.cap / SEG_NNZ + 1;
        Ly.bseg_cap = Ly.n_in + Ly.cap / SEG_NNZ + 1;
        Ly.fslot_cap = Ly.n_in > SEG_NNZ ? 2 * (Ly.cap / SEG_NNZ) + 2 : 0;   // mirror rows <= n_in long
        Ly.bslot_cap = Ly.n_out > SEG_NNZ ? 2 * (Ly.cap / SEG_NNZ) + 2 : 0;  // CSR rows <= n_out long
        Ly.fseg = zalloc<int4>(h, (size_t)Ly.fseg_cap, &rc);
        Ly.bseg = zalloc<int4>(h, (size_t)Ly.bseg_cap, &rc);
        Ly.fmulti = zalloc<int4>(h, (size_t)(Ly.cap / SEG_NNZ + 1), &rc);
        Ly.bmulti = zalloc<int4>(h, (size_t)(Ly.cap / SEG_NNZ + 1), &rc);
        Ly.fws = zalloc<float>(h, (size_t)std::max<int64_t>(Ly.fslot_cap, 1) * CB, &rc);
        Ly.bws = zalloc<float>(h, (size_t)std::max<int64_t>(Ly.bslot_cap, 1) * CB, &rc);
        Ly.bgs = zalloc<float>(h, (size_t)Ly.n_in, &rc);
        Ly.meta = zalloc<LayerMeta>(h, 1, &rc);
        // narrow output layer: stream the canonical rows instead of gathering
        Ly.nout_pad = std::max(2, next_pow2((int)std::min<int64_t>(Ly.n_out, 1 << 20)));
        Ly.narrow = Ly.l == L && Ly.n_out <= NARROW_MAX && (int64_t)Ly.nout_pad * CB <= NARROW_MAX_ELEMS;
        // backward: the row streaming pays for dense-capped rows (all n_L outputs per input row);
        // a sparse output layer's short canonical rows go through the row kernels (C3: 70 -> 19 us)
        Ly.narrow_bwd = Ly.narrow && (Ly.dense || h->narrow_sparse_bwd);
        if (Ly.narrow) {
            Ly.ngrid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)h->num_sms * 4, (Ly.n_in + 63) / 64));
            // CTA partials of a forward pass of up to 128 columns (several forward chunks)
            const int64_t wmax = std::max<int64_t>(CB, std::min<int64_t>(128, NARROW_MAX_ELEMS / Ly.nout_pad));
            Ly.nws = zalloc<float>(h, (size_t)Ly.ngrid * Ly.nout_pad * wmax, &rc);
        }
    }
    if (rc) return rc;
    // --- neuron-layer buffers
    for (int l = 1; l <= L; ++l) {
        const size_t n = (size_t)h->sizes[l - 1];
        // + one zero row after the last chunk: the padding target of the row kernels' gather slots
        h->act[l] = zalloc<float>(h, ((size_t)h->max_chunks_f * n + 1) * h->CBf, &rc);
        if (l >= 2) h->delta[l] = zalloc<float>(h, ((size_t)h->max_chunks * n + 1) * CB, &rc);
        if (l >= 2 && l < L) {
            h->zmask[l] = zalloc<uint4>(h, (size_t)h->max_chunks_f * n, &rc);
            h->kmask[l] = zalloc<uint4>(h, (size_t)h->max_chunks_f * n, &rc);
        }
        h->alive[l] = zalloc<uint8_t>(h, n, &rc);
        if (rc) return rc;
        if (cudaMemsetAsync(h->alive[l], 1, n, h->stream) != cudaSuccess) return set_err(h, SMLP_E_CUDA, "memset");
        h->alive_h[l] = (int64_t)n;
    }
    h->d_err = zalloc<int32_t>(h, 1, &rc);
    // binary-input path of W^(2): bit-packed input, usable when the padded batch fits 128 columns
    if (cfg->input_kind != SMLP_INPUT_REAL && (int64_t)h->max_chunks * CB <= 32 * XBITS_WORDS &&
        (int64_t)h->max_chunks_f * h->CBf <= 32 * XBITS_WORDS) {
        h->xbits = zalloc<uint32_t>(h, (size_t)h->sizes[0] * XBITS_WORDS, &rc);
        h->d_nonbinary = zalloc<int32_t>(h, 1, &rc);
        h->gmirror2 = zalloc<float>(h, (size_t)std::max<int64_t>(h->layers[0].cap, 1), &rc);
    }
    if (cfg->input_kind == SMLP_INPUT_BINARY) {
        if (!h->xbits) return set_err(h, SMLP_E_ARG, "SMLP_INPUT_BINARY needs max_batch <= 128");
        h->input_binary = true;
    }
    {   // implicit delta_{L-1}: a dense-capped 2-output layer on top of a row-kernel hidden layer
        const Layer& Lo = h->layers[L - 2];
        if (h->implicit_delta && L >= 4 && Lo.narrow_bwd && Lo.dense && Lo.nout_pad == 2 && CB <= 64 &&
            !(cfg->dropout > 0.f))
            h->drec = zalloc<uint4>(h, (size_t)h->sizes[L - 2] + 1, &rc);
    }
    h->d_loss = zalloc<float>(h, 1, &rc);
    if (rc) return rc;
    // --- Erdos-Renyi initialisation (R1, R2)
    for (auto& Ly : h->layers) {
        if (Ly.dense) {
            SMLP_TRY(fill_dense_layer(h, Ly));
            continue;
        }
        uint64_t* pos = (uint64_t*)tmp_alloc(h, sizeof(uint64_t) * (size_t)std::max<int64_t>(Ly.cap, 1));
        float* v = (float*)tmp_alloc(h, sizeof(float) * (size_t)std::max<int64_t>(Ly.cap, 1));
        if (!pos || !v) return set_err(h, SMLP_E_NOMEM, "init workspace");
        SMLP_TRY(first_distinct_candidates(h, Ly, P_INIT, 0, Ly.cap, false, nullptr, nullptr,
                                           Ly.n_in * Ly.n_out, pos, v));
        SMLP_TRY(csr_from_sorted_positions(h, Ly, pos, v, Ly.cap));
        tmp_free(h, pos, sizeof(uint64_t) * (size_t)std::max<int64_t>(Ly.cap, 1));
        tmp_free(h, v, sizeof(float) * (size_t)std::max<int64_t>(Ly.cap, 1));
    }
    SMLP_CK(h, cudaStreamSynchronize(h->stream));
    (void)cfg;
    return SMLP_OK;
}

}  // namespace

extern "C" {

const char* sparse_mlp_version(void) { return "sparse_mlp 0.1 (sm_100a)"; }

const char* sparse_mlp_last_error(const smlp_handle* h) {
    return h ? h->err.c_str() : g_create_error.c_str();
}

int sparse_mlp_plan_chunks(const int64_t* sizes, int32_t n_layers, int32_t max_batch, int32_t chunk_batch,
                           int64_t l2_bytes, int32_t* cb, int32_t* cbf) {
    if (!sizes || !cb || !cbf || n_layers < 1 || max_batch < 1 || l2_bytes <= 0)
        return set_err(nullptr, SMLP_E_ARG, "plan_chunks: bad argument");
    if (chunk_batch != 0) {
        if (chunk_batch < 4 || chunk_batch > 128 || (chunk_batch & (chunk_batch - 1)))
            return set_err(nullptr, SMLP_E_ARG, "chunk_batch must be a power of two in [4, 128]");
        *cb = *cbf = chunk_batch;
        return SMLP_OK;
    }
    const double l2 = (double)l2_bytes;
    int64_t nmax = 0;
    for (int l = 0; l < n_layers; ++l) nmax = std::max<int64_t>(nmax, sizes[l]);
    // the widest chunk (<= 128 columns) whose largest activation slab n_l x CB x 4 B fits in the
    // L2, so most row gathers of a pass hit in L2 (C5: 64 columns, 128 MB slabs; measured 6.7
    // ms/step against 7.1 at 32 and 9.3 at 16)
    const int widest = std::min(128, next_pow2(std::max(4, (int)max_batch)));
    int CB = widest;
    while (CB > 4 && (double)nmax * CB * 4.0 > l2) CB >>= 1;
    // forward width: the forward gathers a_{l-1} only (no second operand in flight), so a
    // narrower slab that stays L2-resident pays more than the wider chunk's fewer passes
    // (C5: 32 columns / 64 MB forward, 64 columns / 128 MB backward)
    int CBf = CB;
    while (CBf > 32 && (double)nmax * CBf * 4.0 > 0.5 * l2) CBf >>= 1;
    // layers so wide that not even a 32-column slab fits the L2 (Table 4 widths, >= 1M
    // neurons): the gathers miss either way, so the widest chunk (fewest passes over the
    // indices, longest rows per gather) wins -- T2 / T3 (2.5M / 5M): 9.2 / 18.7 ms at 128
    // columns against 11.1 / 22.5 at 64 and 14.5 / 29.3 at 32
    if (widest >= 32 && (double)nmax * 32 * 4.0 > l2) CB = CBf = widest;
    *cb = CB;
    *cbf = CBf;
    return SMLP_OK;
}

int sparse_mlp_create(const smlp_config* cfg, smlp_handle** out) {
    if (!out) return set_err(nullptr, SMLP_E_ARG, "out is NULL");
    *out = nullptr;
    if (!cfg) return set_err(nullptr, SMLP_E_ARG, "cfg is NULL");
    if (cfg->n_layers < 3 || cfg->n_layers > SMLP_MAX_LAYERS || !cfg->sizes)
        return set_err(nullptr, SMLP_E_ARG, "n_layers must be in [3, 16]");
    for (int l = 0; l < cfg->n_layers; ++l)
        if (cfg->sizes[l] < 1 || cfg->sizes[l] > ((int64_t)1 << 31) - 1)
            return set_err(nullptr, SMLP_E_ARG, "layer " + std::to_string(l + 1) + ": size must be in [1, 2^31)");
    if (!(cfg->epsilon > 0)) return set_err(nullptr, SMLP_E_ARG, "epsilon must be > 0");
    if (!(cfg->alpha >= 0)) return set_err(nullptr, SMLP_E_ARG, "alpha must be >= 0");
    if (!(cfg->dropout >= 0 && cfg->dropout < 1)) return set_err(nullptr, SMLP_E_ARG, "dropout must be in [0, 1)");
    if (cfg->max_batch < 1) return set_err(nullptr, SMLP_E_ARG, "max_batch must be >= 1");
    if (cfg->activation != SMLP_ACT_RELU && cfg->activation != SMLP_ACT_ALL_RELU)
        return set_err(nullptr, SMLP_E_ARG, "unknown activation");
    if (cfg->init < SMLP_INIT_NORMAL || cfg->init > SMLP_INIT_HE_U) return set_err(nullptr, SMLP_E_ARG, "unknown init");
    if (cfg->input_kind != SMLP_INPUT_AUTO && cfg->input_kind != SMLP_INPUT_REAL && cfg->input_kind != SMLP_INPUT_BINARY)
        return set_err(nullptr, SMLP_E_ARG, "unknown input_kind");
    if (cfg->chunk_batch != 0 && (cfg->chunk_batch < 4 || cfg->chunk_batch > 128 || (cfg->chunk_batch & (cfg->chunk_batch - 1))))
        return set_err(nullptr, SMLP_E_ARG, "chunk_batch must be a power of two in [4, 128]");
    if (cudaSetDevice(cfg->device) != cudaSuccess) return set_err(nullptr, SMLP_E_CUDA, "cudaSetDevice failed");
    int l2 = 0;
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, cfg->device);
    if (l2 <= 0) l2 = 126 << 20;
    int CB = 0, CBf = 0;
    if (sparse_mlp_plan_chunks(cfg->sizes, cfg->n_layers, cfg->max_batch, cfg->chunk_batch, l2, &CB, &CBf) != SMLP_OK)
        return SMLP_E_ARG;
    if (const char* e = std::getenv("SMLP_FWD_CB")) CBf = std::atoi(e);
    if (CBf > CB || CBf < 4 || (CBf & (CBf - 1)) || (CBf < CB && CBf < 32))
        return set_err(nullptr, SMLP_E_ARG, "forward chunk width must be a power of two, <= chunk_batch and >= 32 when narrower");

    smlp_handle* h = new smlp_handle();
    h->L = cfg->n_layers;
    for (int l = 0; l < h->L; ++l) h->sizes[l] = cfg->sizes[l];
    h->eps = cfg->epsilon;
    h->activation = cfg->activation;
    h->alpha = cfg->alpha;
    h->dropout = cfg->dropout;
    h->init = cfg->init;
    h->seed = cfg->seed;
    h->rank = cfg->rank;
    h->max_batch = cfg->max_batch;
    h->CB = CB;
    h->max_chunks = (cfg->max_batch + CB - 1) / CB;
    h->CBf = CBf;
    h->max_chunks_f = (cfg->max_batch + CBf - 1) / CBf;
    h->device = cfg->device;
    h->stream = (cudaStream_t)cfg->stream;
    if (cfg->allocator && cfg->allocator->alloc && cfg->allocator->free) {
        h->allocator = *cfg->allocator;
        h->has_allocator = true;
    }
    cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, cfg->device);
    if (const char* e = std::getenv("SMLP_IMPLICIT_DELTA")) h->implicit_delta = std::atoi(e) != 0;
    if (const char* e = std::getenv("SMLP_NARROW_SPARSE_BWD")) h->narrow_sparse_bwd = std::atoi(e) != 0;
    if (const char* e = std::getenv("SMLP_SHORT_MAX_FWD")) h->short_max_fwd = std::atoi(e);
    if (const char* e = std::getenv("SMLP_SHORT_MAX_BWD")) h->short_max_bwd = std::atoi(e);
    if (const char* e = std::getenv("SMLP_SHORT_MIN_ROWS")) h->short_min_rows = std::atoll(e);
    const int rc = build_handle(h, cfg);
    if (rc != SMLP_OK) {
        g_create_error = h->err;
        sparse_mlp_destroy(h);
        return rc;
    }
    *out = h;
    return SMLP_OK;
}

int sparse_mlp_destroy(smlp_handle* h) {
    if (!h) return SMLP_OK;
    cudaStreamSynchronize(h->stream);
    for (auto& r : h->prof_recs) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    for (auto e : h->ev_pool) cudaEventDestroy(e);
    for (auto& a : h->allocs) tmp_free(h, a.ptr, a.bytes);
    h->allocs.clear();
    for (auto e : h->layer_ev)
        if (e) cudaEventDestroy(e);
    for (int k = 0; k < 2; ++k) {
        if (h->ev_copied[k]) cudaEventDestroy(h->ev_copied[k]);
        if (h->ev_consumed[k]) cudaEventDestroy(h->ev_consumed[k]);
    }
    if (h->copy_stream) {
        cudaStreamSynchronize(h->copy_stream);
        cudaStreamDestroy(h->copy_stream);
    }
    if (h->aux_stream) {
        cudaStreamSynchronize(h->aux_stream);
        cudaStreamDestroy(h->aux_stream);
    }
    for (auto e : h->aux_ev)
        if (e) cudaEventDestroy(e);
    cudaStreamSynchronize(h->stream);
    delete h;
    return SMLP_OK;
}

int sparse_mlp_profile(smlp_handle* h, int32_t enable) {
    if (!h) return SMLP_E_ARG;
    if (enable) {
        for (auto& r : h->prof_recs) {
            h->ev_pool.push_back(r.a);
            h->ev_pool.push_back(r.b);
        }
        h->prof_recs.clear();
    }
    h->prof = enable != 0;
    return SMLP_OK;
}

int sparse_mlp_profile_read(smlp_handle* h, smlp_kernel_stat* out, int32_t cap, int32_t* n) {
    if (!h || !n) return SMLP_E_ARG;
    SMLP_CK(h, cudaStreamSynchronize(h->stream));
    std::vector<smlp_kernel_stat> agg;
    for (auto& r : h->prof_recs) {
        float ms = 0.f;
        SMLP_CK(h, cudaEventElapsedTime(&ms, r.a, r.b));
        smlp_kernel_stat* s = nullptr;
        for (auto& a : agg)
            if (a.kind == r.kind && a.layer == r.layer) s = &a;
        if (!s) {
            agg.push_back(smlp_kernel_stat{r.kind, r.layer, 0, 0.0, 0.0, 0.0});
            s = &agg.back();
        }
        // running mean of the per-launch algorithmic figures (chunks may differ in width)
        s->bytes_per_launch = (s->bytes_per_launch * (double)s->launches + r.bytes) / (double)(s->launches + 1);
        s->flops_per_launch = (s->flops_per_launch * (double)s->launches + r.flops) / (double)(s->launches + 1);
        s->launches += 1;
        s->total_ms += ms;
    }
    *n = (int32_t)agg.size();
    for (int32_t k = 0; k < std::min<int32_t>(cap, *n); ++k) out[k] = agg[(size_t)k];
    return SMLP_OK;
}

int sparse_mlp_params_updated(smlp_handle* h) {
    if (!h) return SMLP_E_ARG;
    for (auto& Ly : h->layers) SMLP_TRY(refresh_mirror_values(h, Ly));
    return SMLP_OK;
}

int sparse_mlp_set_step_counter(smlp_handle* h, const uint64_t* dev_counter) {
    if (!h) return SMLP_E_ARG;
    h->step_counter = dev_counter;
    return SMLP_OK;
}

int sparse_mlp_set_stream(smlp_handle* h, void* stream) {
    if (!h) return SMLP_E_ARG;
    h->stream = (cudaStream_t)stream;
    return SMLP_OK;
}

int sparse_mlp_forward(smlp_handle* h, const float* x, const int32_t* x_idx, int32_t B, int32_t train, uint64_t step,
                       float* probs) {
    if (!h) return SMLP_E_ARG;
    if (!x) return set_err(h, SMLP_E_ARG, "x is NULL");
    if (B < 1 || B > h->max_batch)
        return set_err(h, SMLP_E_SHAPE, "layer 1: B=" + std::to_string(B) + " > max_batch=" + std::to_string(h->max_batch));
    return run_forward(h, x, x_idx, B, train != 0, step, probs);
}

int sparse_mlp_backward(smlp_handle* h, const int32_t* labels, const int32_t* y_idx, float* loss,
                        const smlp_sgd* fused) {
    if (!h) return SMLP_E_ARG;
    if (!labels) return set_err(h, SMLP_E_ARG, "labels is NULL");
    if (!h->trace_valid || !h->trace_train || h->trace_version != h->version)
        return set_err(h, SMLP_E_STALE, "backward needs a train-mode forward on the current topology version");
    int rc;
    if (fused) {
        // measured faster than applying Eq. 1 inside the last chunk's backward: the
        // backward only accumulates the gradient (the last chunk of a large model into grad2),
        // then one streaming Eq. 1 pass over the whole view (grad_scale 1) and the mirror refresh
        smlp_sgd f = *fused;
        f.grad_scale = 1.f;
        rc = run_backward_step(h, labels, y_idx, loss, &f);
    } else {
        rc = run_backward_step(h, labels, y_idx, loss, nullptr);
    }
    if (rc == SMLP_OK) {
        h->grads_pending = fused == nullptr;
        h->trace_valid = false;   // the trace is consumed (and fused updates changed the weights)
    }
    return rc;
}

int sparse_mlp_step(smlp_handle* h, const smlp_sgd* sgd) {
    if (!h || !sgd) return SMLP_E_ARG;
    if (!h->grads_pending) return set_err(h, SMLP_E_STATE, "step without pending gradients");
    const int rc = run_step(h, sgd);
    if (rc == SMLP_OK) h->grads_pending = false;
    return rc;
}

// pipelined host-buffer step: staging buffer k = call parity; its H2D runs on the copy stream
// (waiting only for the forward that last read buffer k, two calls ago), so the copy of step s+1
// overlaps the compute of step s
static int stage_and_step(smlp_handle* h, const float* x_host, const int32_t* y_host, int32_t B, uint64_t step,
                          const smlp_sgd* sgd, float* loss_host) {
    if (!h || !x_host || !y_host || !sgd) return SMLP_E_ARG;
    if (B < 1 || B > h->max_batch) return set_err(h, SMLP_E_SHAPE, "B out of range");
    if (!h->x_stage[0]) {
        for (int k = 0; k < 2; ++k) {
            h->x_stage[k] = (float*)dev_alloc(h, sizeof(float) * (size_t)h->max_batch * (size_t)h->sizes[0]);
            h->y_stage[k] = (int32_t*)dev_alloc(h, sizeof(int32_t) * (size_t)h->max_batch);
            if (!h->x_stage[k] || !h->y_stage[k]) return set_err(h, SMLP_E_NOMEM, "staging buffers");
            SMLP_CK(h, cudaEventCreateWithFlags(&h->ev_copied[k], cudaEventDisableTiming));
            SMLP_CK(h, cudaEventCreateWithFlags(&h->ev_consumed[k], cudaEventDisableTiming));
            SMLP_CK(h, cudaEventRecord(h->ev_consumed[k], h->stream));
        }
        SMLP_CK(h, cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking));
    }
    const int k = h->stage_idx;
    h->stage_idx ^= 1;
    SMLP_CK(h, cudaStreamWaitEvent(h->copy_stream, h->ev_consumed[k], 0));
    SMLP_CK(h, cudaMemcpyAsync(h->x_stage[k], x_host, sizeof(float) * (size_t)B * (size_t)h->sizes[0],
                               cudaMemcpyHostToDevice, h->copy_stream));
    SMLP_CK(h, cudaMemcpyAsync(h->y_stage[k], y_host, sizeof(int32_t) * (size_t)B, cudaMemcpyHostToDevice,
                               h->copy_stream));
    SMLP_CK(h, cudaEventRecord(h->ev_copied[k], h->copy_stream));
    SMLP_CK(h, cudaStreamWaitEvent(h->stream, h->ev_copied[k], 0));
    SMLP_TRY(sparse_mlp_forward(h, h->x_stage[k], nullptr, B, 1, step, nullptr));
    SMLP_CK(h, cudaEventRecord(h->ev_consumed[k], h->stream));
    smlp_sgd f = *sgd;
    f.grad_scale = 1.f;
    SMLP_TRY(sparse_mlp_backward(h, h->y_stage[k], nullptr, h->d_loss, &f));
    if (loss_host) SMLP_CK(h, cudaMemcpyAsync(loss_host, h->d_loss, sizeof(float), cudaMemcpyDeviceToHost, h->stream));
    return SMLP_OK;
}

int sparse_mlp_train_step_host(smlp_handle* h, const float* x_host, const int32_t* y_host, int32_t B, uint64_t step,
                               const smlp_sgd* sgd, float* loss_host) {
    SMLP_TRY(stage_and_step(h, x_host, y_host, B, step, sgd, loss_host));
    SMLP_CK(h, cudaStreamSynchronize(h->stream));
    return SMLP_OK;
}

int sparse_mlp_train_step_host_async(smlp_handle* h, const float* x_host, const int32_t* y_host, int32_t B,
                                     uint64_t step, const smlp_sgd* sgd, float* loss_host) {
    return stage_and_step(h, x_host, y_host, B, step, sgd, loss_host);
}

int sparse_mlp_join(smlp_handle* h) {
    // every call joins its side-stream work (mirror refreshes) before returning: nothing pending
    return h ? SMLP_OK : SMLP_E_ARG;
}

int sparse_mlp_sync(smlp_handle* h) {
    if (!h) return SMLP_E_ARG;
    SMLP_CK(h, cudaStreamSynchronize(h->stream));
    return check_data_flag(h);
}

int sparse_mlp_wait_layer(smlp_handle* h, int32_t l, void* stream) {
    if (!h || l < 2 || l > h->L) return SMLP_E_ARG;
    if (!h->layer_ev[l]) return set_err(h, SMLP_E_STATE, "no backward recorded for this layer");
    SMLP_CK(h, cudaStreamWaitEvent((cudaStream_t)stream, h->layer_ev[l], 0));
    return SMLP_OK;
}

int sparse_mlp_view_layout(smlp_handle* h, int64_t* val_off, int64_t* cap, int64_t* bias_base) {
    if (!h) return SMLP_E_ARG;
    for (int l = 2; l <= h->L; ++l) {
        const smlp::Layer& Ly = h->layers[l - 2];
        if (val_off) val_off[l - 2] = Ly.val_off;
        if (cap) cap[l - 2] = Ly.cap;
    }
    if (bias_base) *bias_base = h->bias_base;
    return SMLP_OK;
}

int sparse_mlp_grad_view(smlp_handle* h, float** dev, int64_t* count, uint64_t* version) {
    if (!h) return SMLP_E_ARG;
    if (dev) *dev = h->grad;
    if (count) *count = h->param_count;
    if (version) *version = h->version;
    return SMLP_OK;
}

int sparse_mlp_param_view(smlp_handle* h, float** dev, int64_t* count, uint64_t* version) {
    if (!h) return SMLP_E_ARG;
    if (dev) *dev = h->param;
    if (count) *count = h->param_count;
    if (version) *version = h->version;
    return SMLP_OK;
}

int sparse_mlp_evolve_topology(smlp_handle* h, double zeta, uint64_t evolve_idx, int64_t* removed_per_layer) {
    if (!h) return SMLP_E_ARG;
    if (!(zeta > 0.0 && zeta < 1.0)) return set_err(h, SMLP_E_ARG, "zeta must be in (0, 1)");
    SMLP_TRY(check_data_flag(h));
    return run_evolve(h, zeta, evolve_idx, removed_per_layer);
}

int sparse_mlp_prune_neurons(smlp_handle* h, double percentile, int32_t flags, int64_t* pruned_per_layer,
                             int64_t* removed_conn) {
    if (!h) return SMLP_E_ARG;
    if (!(percentile >= 0.0 && percentile < 100.0)) return set_err(h, SMLP_E_ARG, "percentile must be in [0, 100)");
    SMLP_TRY(check_data_flag(h));
    return run_prune(h, percentile, flags, pruned_per_layer, removed_conn);
}

int sparse_mlp_importance(smlp_handle* h, int32_t l, double* out, int32_t to_host) {
    if (!valid_layer(h, l, 2) || l == h->L) return h ? set_err(h, SMLP_E_SHAPE, "importance: hidden layer 2..L-1") : SMLP_E_ARG;
    if (!out) return set_err(h, SMLP_E_ARG, "out is NULL");
    const size_t n = (size_t)h->sizes[l - 1];
    double* dst = out;
    if (to_host) {
        dst = (double*)tmp_alloc(h, n * sizeof(double));
        if (!dst) return set_err(h, SMLP_E_NOMEM, "importance buffer");
    }
    SMLP_TRY(run_importance(h, l, dst));
    if (to_host) {
        SMLP_CK(h, cudaMemcpyAsync(out, dst, n * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
        SMLP_CK(h, cudaStreamSynchronize(h->stream));
        tmp_free(h, dst, n * sizeof(double));
    } else {
        SMLP_CK(h, cudaStreamSynchronize(h->stream));
    }
    return SMLP_OK;
}

int sparse_mlp_info(smlp_handle* h, smlp_info* info) {
    if (!h || !info) return SMLP_E_ARG;
    std::memset(info, 0, sizeof(*info));
    info->n_layers = h->L;
    info->chunk_batch = h->CB;
    info->fwd_chunk_batch = h->CBf;
    info->version = h->version;
    for (int l = 1; l <= h->L; ++l) {
        info->sizes[l - 1] = h->sizes[l - 1];
        info->alive[l - 1] = h->alive_h[l];
    }
    for (auto& Ly : h->layers) {
        info->nnz[Ly.l - 1] = Ly.nnz;
        info->cap[Ly.l - 1] = Ly.cap;
        info->dense_capped[Ly.l - 1] = Ly.dense ? 1 : 0;
        info->val_offset[Ly.l - 1] = Ly.val_off;
        info->bias_offset[Ly.l - 1] = Ly.bias_off;
    }
    info->param_count = h->param_count;
    info->launches = h->launches;
    info->implicit_delta = h->drec ? 1 : 0;
    return SMLP_OK;
}

int sparse_mlp_export_layer(smlp_handle* h, int32_t l, int32_t* row_ptr, int32_t* col_idx, float* val, float* mom,
                            int32_t to_host) {
    if (!valid_layer(h, l, 2)) return h ? set_err(h, SMLP_E_SHAPE, "export_layer: l must be in 2..L") : SMLP_E_ARG;
    const Layer& Ly = h->layers[(size_t)(l - 2)];
    const cudaMemcpyKind k = to_host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    const size_t nz = (size_t)Ly.nnz;
    if (row_ptr) SMLP_CK(h, cudaMemcpyAsync(row_ptr, Ly.row_ptr, sizeof(int32_t) * ((size_t)Ly.n_in + 1), k, h->stream));
    if (col_idx && nz) SMLP_CK(h, cudaMemcpyAsync(col_idx, Ly.col, sizeof(int32_t) * nz, k, h->stream));
    if (val && nz) SMLP_CK(h, cudaMemcpyAsync(val, Ly.val, sizeof(float) * nz, k, h->stream));
    if (mom && nz) SMLP_CK(h, cudaMemcpyAsync(mom, Ly.mom, sizeof(float) * nz, k, h->stream));
    SMLP_CK(h, cudaStreamSynchronize(h->stream));
    return SMLP_OK;
}

int sparse_mlp_import_layer(smlp_handle* h, int32_t l, int64_t nnz, const int32_t* row_ptr, const int32_t* col_idx,
                            const float* val, const float* mom) {
    if (!valid_layer(h, l, 2)) return h ? set_err(h, SMLP_E_SHAPE, "import_layer: l must be in 2..L") : SMLP_E_ARG;
    Layer& Ly = h->layers[(size_t)(l - 2)];
    if (!row_ptr || (nnz > 0 && (!col_idx || !val))) return set_err(h, SMLP_E_ARG, "import_layer: NULL array");
    if (nnz < 0 || nnz > Ly.cap) return set_err(h, SMLP_E_SHAPE, "import_layer: nnz exceeds the layer capacity");
    // invariants of SPEC S:26-29
    if (row_ptr[0] != 0 || row_ptr[Ly.n_in] != nnz) return set_err(h, SMLP_E_STRUCT, "import_layer: row_ptr ends");
    for (int64_t i = 0; i < Ly.n_in; ++i) {
        if (row_ptr[i + 1] < row_ptr[i])
            return set_err(h, SMLP_E_STRUCT, "import_layer: row_ptr decreasing at row " + std::to_string(i));
        for (int32_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
            const int32_t c = col_idx[k];
            if (c < 0 || c >= Ly.n_out || (k > row_ptr[i] && col_idx[k - 1] >= c))
                return set_err(h, SMLP_E_STRUCT, "import_layer: invalid entry at (row " + std::to_string(i) +
                                                     ", col " + std::to_string(c) + ")");
        }
    }
    const size_t nz = (size_t)nnz;
    SMLP_CK(h, cudaMemcpyAsync(Ly.row_ptr, row_ptr, sizeof(int32_t) * ((size_t)Ly.n_in + 1), cudaMemcpyHostToDevice,
                               h->stream));
    if (nz) {
        SMLP_CK(h, cudaMemcpyAsync(Ly.col, col_idx, sizeof(int32_t) * nz, cudaMemcpyHostToDevice, h->stream));
        SMLP_CK(h, cudaMemcpyAsync(Ly.val, val, sizeof(float) * nz, cudaMemcpyHostToDevice, h->stream));
        if (mom) SMLP_CK(h, cudaMemcpyAsync(Ly.mom, mom, sizeof(float) * nz, cudaMemcpyHostToDevice, h->stream));
        else SMLP_CK(h, cudaMemsetAsync(Ly.mom, 0, sizeof(float) * nz, h->stream));
    }
    SMLP_TRY(zero_tail(h, Ly, nnz));
    Ly.nnz = nnz;
    SMLP_TRY(rebuild_derived(h, Ly));
    h->version++;
    h->trace_valid = false;
    return SMLP_OK;
}

int sparse_mlp_export_bias(smlp_handle* h, int32_t l, float* bias, float* bias_mom) {
    if (!valid_layer(h, l, 2)) return h ? set_err(h, SMLP_E_SHAPE, "export_bias: l must be in 2..L") : SMLP_E_ARG;
    const Layer& Ly = h->layers[(size_t)(l - 2)];
    const size_t n = (size_t)Ly.n_out;
    if (bias) SMLP_CK(h, cudaMemcpyAsync(bias, Ly.bias, n * 4, cudaMemcpyDeviceToHost, h->stream));
    if (bias_mom) SMLP_CK(h, cudaMemcpyAsync(bias_mom, Ly.bias_mom, n * 4, cudaMemcpyDeviceToHost, h->stream));
    SMLP_CK(h, cudaStreamSynchronize(h->stream));
    return SMLP_OK;
}

int sparse_mlp_import_bias(smlp_handle* h, int32_t l, const float* bias, const float* bias_mom) {
    if (!valid_layer(h, l, 2)) return h ? set_err(h, SMLP_E_SHAPE, "import_bias: l must be in 2..L") : SMLP_E_ARG;
    const Layer& Ly = h->layers[(size_t)(l - 2)];
    const size_t n = (size_t)Ly.n_out;
    if (bias) SMLP_CK(h, cudaMemcpyAsync(Ly.bias, bias, n * 4, cudaMemcpyHostToDevice, h->stream));
    if (bias_mom) SMLP_CK(h, cudaMemcpyAsync(Ly.bias_mom, bias_mom, n * 4, cudaMemcpyHostToDevice, h->stream));
    SMLP_CK(h, cudaStreamSynchronize(h->stream));
    return SMLP_OK;
}

int sparse_mlp_export_alive(smlp_handle* h, int32_t l, uint8_t* alive) {
    if (!valid_layer(h, l, 1) || !alive) return h ? set_err(h, SMLP_E_SHAPE, "export_alive: bad layer") : SMLP_E_ARG;
    SMLP_CK(h, cudaMemcpyAsync(alive, h->alive[l], (size_t)h->sizes[l - 1], cudaMemcpyDeviceToHost, h->stream));
    SMLP_CK(h, cudaStreamSynchronize(h->stream));
    return SMLP_OK;
}

int sparse_mlp_import_alive(smlp_handle* h, int32_t l, const uint8_t* alive) {
    if (!valid_layer(h, l, 1) || !alive) return h ? set_err(h, SMLP_E_SHAPE, "import_alive: bad layer") : SMLP_E_ARG;
    const size_t n = (size_t)h->sizes[l - 1];
    std::vector<uint8_t> a(alive, alive + n);
    int64_t cnt = 0;
    for (auto& v : a) {
        v = v ? 1 : 0;
        cnt += v;
    }
    SMLP_CK(h, cudaMemcpyAsync(h->alive[l], a.data(), n, cudaMemcpyHostToDevice, h->stream));
    SMLP_CK(h, cudaStreamSynchronize(h->stream));
    h->alive_h[l] = cnt;
    h->version++;
    h->trace_valid = false;
    return SMLP_OK;
}

int sparse_mlp_export_trace(smlp_handle* h, int32_t kind, int32_t l, float* out) {
    if (!h || !out) return SMLP_E_ARG;
    if (kind == 0 || kind == 1) {
        const int CB = kind == 0 ? h->CBf : h->CB;   // act: forward layout, delta: backward layout
        if (!valid_layer(h, l, kind == 0 ? 1 : 2)) return set_err(h, SMLP_E_SHAPE, "export_trace: bad layer");
        const int B = h->trace_B;
        if (B < 1) return set_err(h, SMLP_E_STATE, "export_trace: no forward yet");
        const int nchunks = (B + CB - 1) / CB;
        const int64_t n = h->sizes[l - 1];
        std::vector<float> raw((size_t)nchunks * (size_t)n * CB);
        const float* src = kind == 0 ? h->act[l] : h->delta[l];
        SMLP_CK(h, cudaMemcpyAsync(raw.data(), src, raw.size() * 4, cudaMemcpyDeviceToHost, h->stream));
        SMLP_CK(h, cudaStreamSynchronize(h->stream));
        for (int b = 0; b < B; ++b) {
            const int c = b / CB, lb = b % CB;
            for (int64_t j = 0; j < n; ++j) out[(int64_t)b * n + j] = raw[((size_t)c * n + j) * CB + lb];
        }
        return SMLP_OK;
    }
    if (kind == 2 || kind == 3) {
        if (!valid_layer(h, l, 2)) return set_err(h, SMLP_E_SHAPE, "export_trace: bad layer");
        const Layer& Ly = h->layers[(size_t)(l - 2)];
        const float* src = kind == 2 ? Ly.grad : Ly.bias_grad;
        const size_t n = kind == 2 ? (size_t)Ly.nnz : (size_t)Ly.n_out;
        if (n) SMLP_CK(h, cudaMemcpyAsync(out, src, n * 4, cudaMemcpyDeviceToHost, h->stream));
        SMLP_CK(h, cudaStreamSynchronize(h->stream));
        return SMLP_OK;
    }
    if (kind == 4) {   // path flag of the last forward: binary-input W^(2) path taken (1), not (0), off (-1)
        if (!h->xbits) {
            out[0] = -1.f;
            return SMLP_OK;
        }
        int32_t nb = 0;
        SMLP_CK(h, cudaMemcpyAsync(&nb, h->d_nonbinary, 4, cudaMemcpyDeviceToHost, h->stream));
        SMLP_CK(h, cudaStreamSynchronize(h->stream));
        out[0] = nb ? 0.f : 1.f;
        return SMLP_OK;
    }
    return set_err(h, SMLP_E_ARG, "export_trace: unknown kind");
}

}  // extern "C"
