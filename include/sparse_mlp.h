/*
 * sparse_mlp.h — C ABI of libsparse_mlp.so, the B200 (sm_100a) hot path of truly sparse
 * MLP training with SET, All-ReLU and Importance Pruning (arXiv 2102.01732).
 *
 * Citations: "PAPER.md:n" = line n of the paper text; readings R1..R26 = DESIGN.md
 * "Readings of the paper".  The problem statement the calls follow:
 *   - train f_s(x; theta_s) with sparse W^(l), n_{l-1} x n_l, w_ij = 0 meaning "no
 *     connection", to minimise sum L(f(x; theta), y)
 *   - Alg. 2 init / train / update / prune / evolve loop
 *   - Alg. 1 gradient exchange and model averaging
 *
 * Conventions (every call):
 *   - Return 0 (SMLP_OK) on success, a negative SMLP_E_* code on failure; the text of the
 *     last failure is sparse_mlp_last_error(h).  No call ever falls back to the CPU.
 *   - Asynchrony: calls enqueue work on the handle's stream (create's cfg.stream, or the
 *     one set by sparse_mlp_set_stream) and return immediately unless marked SYNC.
 *   - Ownership: the caller owns every pointer it passes (x, labels, probs, loss, host
 *     arrays) and keeps it valid until the stream's work completes.  The library owns all
 *     model state and workspace, allocated through cfg.allocator (or cudaMallocAsync).
 *   - Graph capture: forward / backward / step / train_step_device do no host sync and no
 *     allocation once the handle exists, and keep every device pointer stable across
 *     evolve_topology / prune_neurons (device-side counts), so a CUDA graph captured once
 *     stays valid for the life of the handle (per batch size B).
 *   - Threading: not thread-safe per handle; callers serialise.
 *   - Layer indices follow the paper: neuron layers l = 1..L (input l = 1),
 *     weight layer l = 2..L is W^(l) between neuron layers l-1 and l.
 */
#ifndef SPARSE_MLP_H
#define SPARSE_MLP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SMLP_MAX_LAYERS 16

/* status codes */
#define SMLP_OK        0
#define SMLP_E_ARG    -1   /* invalid argument / configuration (S:119 preconditions)        */
#define SMLP_E_NOMEM  -2   /* allocator returned NULL                                        */
#define SMLP_E_CUDA   -3   /* a CUDA runtime call or kernel launch failed                    */
#define SMLP_E_SHAPE  -4   /* B > max_batch, layer index out of range, buffer too small      */
#define SMLP_E_STALE  -5   /* backward without a train-mode forward on the current topology  */
#define SMLP_E_DATA   -6   /* a label outside [0, n_L) was seen by a previous backward       */
#define SMLP_E_STATE  -7   /* step without pending gradients                                 */
#define SMLP_E_STRUCT -8   /* imported CSR violates the invariants (sorted unique, bounds)  */

/* activation (Eq. 3 All-ReLU PAPER.md:106-112; Eq. 5 ReLU PAPER.md:533-539) */
#define SMLP_ACT_RELU      0
#define SMLP_ACT_ALL_RELU  1

/* weight initialisation (Table 5 names; reading R3) */
#define SMLP_INIT_NORMAL     0   /* N(0, 2/n_{l-1}), Box-Muller                          */
#define SMLP_INIT_XAVIER_U   1   /* U(-sqrt(6/(n_{l-1}+n_l)), +sqrt(6/(n_{l-1}+n_l)))    */
#define SMLP_INIT_HE_U       2   /* U(-sqrt(6/n_{l-1}), +sqrt(6/n_{l-1}))                */

/* input kinds (smlp_config.input_kind) */
#define SMLP_INPUT_AUTO 0
#define SMLP_INPUT_REAL 1
#define SMLP_INPUT_BINARY 2   /* inputs promised {0,1} (needs max_batch <= 128): as AUTO, and a
                                 batch that breaks the promise is reported -- SMLP_E_DATA at the
                                 next synchronising call.  That batch's step is still computed
                                 correctly, through the fp32 layer-2 kernels (they run whenever
                                 the staged batch is not binary), so nothing is corrupted      */

/* prune flags */
#define SMLP_PRUNE_OUTGOING  1   /* also remove the outgoing row of a pruned neuron (R17)   */

typedef struct smlp_handle smlp_handle;

/* Device allocator.  alloc(bytes, stream, ctx) returns device memory or NULL; free(ptr,
 * bytes, stream, ctx) releases it.  Used for every model / workspace allocation.  The
 * Python binding passes torch's caching allocator.  NULL => cudaMallocAsync/cudaFreeAsync. */
typedef struct {
    void* (*alloc)(size_t bytes, void* stream, void* ctx);
    void  (*free)(void* ptr, size_t bytes, void* stream, void* ctx);
    void* ctx;
} smlp_allocator;

typedef struct {
    int32_t        n_layers;     /* L >= 3 (input, >= 1 hidden, output)                       */
    const int64_t* sizes;        /* [L] neuron counts n_1..n_L, each >= 1 (host pointer)      */
    double         epsilon;      /* ER density parameter eps > 0             */
    int32_t        activation;   /* SMLP_ACT_*                                                */
    float          alpha;        /* All-ReLU slope alpha >= 0                                 */
    float          dropout;      /* inverted dropout rate in [0, 1) on hidden activations     */
    int32_t        init;         /* SMLP_INIT_*                                               */
    uint64_t       seed;         /* Philox key: topology and values are a function of it      */
    int32_t        rank;         /* data-parallel rank: enters the dropout stream only        */
    int32_t        max_batch;    /* largest B passed to forward, >= 1                         */
    int32_t        chunk_batch;  /* batch columns per activation chunk (4..128, power of 2);
                                    0 = auto: min(128, next_pow2(max(4, max_batch))), halved
                                    while the widest layer's slab n_l x CB x 4 B exceeds the
                                    L2; the forward tensors (a_l, masks) then use their own
                                    width CBf <= CB, halved (not below 32) while the slab
                                    exceeds half the L2; if not even a 32-column slab fits
                                    the L2, CB = CBf = the widest.  Explicit: CBf = CB.  Env
                                    SMLP_FWD_CB overrides CBf (power of 2, <= CB, >= 32 if
                                    narrower; else SMLP_E_ARG)                               */
    int32_t        device;       /* CUDA device ordinal                                       */
    void*          stream;       /* cudaStream_t the handle enqueues on (NULL = legacy)       */
    const smlp_allocator* allocator; /* NULL = cudaMallocAsync on `stream`                   */
    int32_t        input_kind;   /* SMLP_INPUT_AUTO: detect {0,1}-only batches on the device and
                                    take the bit-packed W^(2) path for them (needs max_batch
                                    <= 128); SMLP_INPUT_REAL: inputs are real-valued, no
                                    detection and no bit path (4 fewer launches per step);
                                    SMLP_INPUT_BINARY: see the define                        */
} smlp_config;

/* Momentum SGD with weight decay, Eq. 1 in velocity form (reading R14):
 *   v <- mu v - lr (grad_scale g + weight_decay w);  w <- w + v;   biases: no decay.      */
typedef struct {
    float lr;
    float momentum;
    float weight_decay;
    float grad_scale;   /* 1/K after a K-rank SUM allreduce; 1 for one rank */
} smlp_sgd;

typedef struct {
    int32_t  n_layers;
    int32_t  chunk_batch;
    uint64_t version;                        /* topology version, +1 per structural edit  */
    int64_t  sizes[SMLP_MAX_LAYERS];         /* n_l at index l-1                          */
    int64_t  alive[SMLP_MAX_LAYERS];         /* alive neurons of layer l at index l-1     */
    int64_t  nnz[SMLP_MAX_LAYERS];           /* nnz of W^(l) at index l-1 (0 for l = 1)   */
    int64_t  cap[SMLP_MAX_LAYERS];           /* capacity of W^(l) (initial nnz)           */
    int32_t  dense_capped[SMLP_MAX_LAYERS];  /* W^(l) dense-capped, never evolved (R9)    */
    int64_t  val_offset[SMLP_MAX_LAYERS];    /* offset of W^(l) values in the param view  */
    int64_t  bias_offset[SMLP_MAX_LAYERS];   /* offset of b_l in the param view           */
    int64_t  param_count;                    /* floats in the param / grad views          */
    int64_t  launches;                       /* kernels launched by this handle so far    */
    int32_t  fwd_chunk_batch;                /* CBf: chunk width of a_l and the masks     */
    int32_t  implicit_delta;                 /* 1: the backward of W^(L-1) recomputes delta_{L-1}
                                                from per-neuron records (dense-capped 2-output
                                                W^(L), chunk_batch <= 64, no dropout) instead of
                                                gathering it; results are bit-identical           */
} smlp_info;

/* sparse_mlp_create — PAPER.md:51-52 ("Initially each W^(l) is a Erdos-Renyi random graph"),
 * Alg. 2 PAPER.md:643-646.  Per weight layer M = min(n_in n_out, floor(eps (n_in + n_out)))
 * connections (R1): the first M distinct positions of the INIT Philox stream (R2), values
 * from the scheme `init`; dense-capped layers take every position.  Momentum and biases are
 * zero, version = 0.  SYNC (returns after the initial topology is built).
 * Errors: SMLP_E_ARG (L < 3 or > SMLP_MAX_LAYERS, n_l < 1, eps <= 0, alpha < 0, dropout
 * outside [0,1), max_batch < 1, bad enum, nnz >= 2^31 in a layer), SMLP_E_NOMEM, SMLP_E_CUDA.
 * On failure *out is NULL. */
int sparse_mlp_create(const smlp_config* cfg, smlp_handle** out);

/* sparse_mlp_plan_chunks — the chunk widths sparse_mlp_create picks (host only, no device call;
 * DESIGN.md §4-5).  sizes[n_layers] = n_1..n_L, l2_bytes = the device's L2 size.  chunk_batch
 * != 0: *cb = *cbf = chunk_batch.  0 (auto): *cb = the widest power of two <= min(128,
 * next_pow2(max(4, max_batch))) whose widest slab n_l x cb x 4 B fits the L2; *cbf = cb halved
 * (not below 32) while the slab exceeds half the L2; if not even a 32-column slab fits the L2,
 * *cb = *cbf = the widest.  (create then applies the SMLP_FWD_CB override.)
 * Errors: SMLP_E_ARG (NULL pointer, n_layers < 1, max_batch < 1, l2_bytes <= 0, chunk_batch
 * not 0 or a power of two in [4, 128]). */
int sparse_mlp_plan_chunks(const int64_t* sizes, int32_t n_layers, int32_t max_batch, int32_t chunk_batch,
                           int64_t l2_bytes, int32_t* cb, int32_t* cbf);

/* Frees everything through the allocator on the handle's stream.  NULL is a no-op. */
int sparse_mlp_destroy(smlp_handle* h);

/* Replace the stream subsequent calls enqueue on (e.g. torch's current stream).  When the stream
 * changes, pending side-stream work (deferred mirror refreshes, SMLP_DEFER_MIRROR) is first joined
 * on the old one.  Errors: SMLP_E_ARG (NULL handle), SMLP_E_CUDA. */
int sparse_mlp_set_stream(smlp_handle* h, void* stream);

/* sparse_mlp_forward — a_1 = x; for l = 2..L: z_l = a_{l-1} W^(l) + b_l; for hidden l,
 * a_l = f_l(z_l) (Eq. 3) then, if train, inverted dropout with rate
 * cfg.dropout drawn from Philox(DROPOUT, rank, l, step) (R13); p = softmax(z_L).
 *   x:      device fp32, row-major [rows x n_1]; sample b is row (x_idx ? x_idx[b] : b).
 *   x_idx:  device int32 [B] or NULL.
 *   B:      1..max_batch.   train: 0/1.   step: global step (dropout stream counter).
 *   probs:  device fp32 [B x n_L] row-major, or NULL.
 * Records a trace (version, B, train) for backward.
 * Errors: SMLP_E_SHAPE (B < 1 or B > max_batch), SMLP_E_CUDA. */
int sparse_mlp_forward(smlp_handle* h, const float* x, const int32_t* x_idx, int32_t B,
                       int32_t train, uint64_t step, float* probs);

/* sparse_mlp_backward — softmax cross-entropy (R12): loss = (1/B) sum_b -ln p[b, y_b],
 * delta_L = (p - onehot)/B; for l = L..2: g_ij = sum_b a_{l-1}[b,i] delta_l[b,j] on the
 * support only (SDDMM), gb_l = sum_b delta_l[b,:], and for l >= 3
 * delta_{l-1} = (delta_l W^(l)T) * f'_{l-1}(z_{l-1}) * keep/(1-r).
 *   labels: device int32 [rows]; sample b uses labels[y_idx ? y_idx[b] : b].
 *   y_idx:  device int32 [B] or NULL (normally the x_idx of the forward).
 *   loss:   device fp32 scalar or NULL.
 *   fused:  NULL -> gradients are written to the grad view for a later sparse_mlp_step
 *           (the multi-GPU path, after the caller's allreduce); non-NULL -> the Eq. 1
 *           update (fused->grad_scale ignored, = 1) is applied in the same pass.
 * Errors: SMLP_E_STALE (no train-mode forward since the last topology change),
 * SMLP_E_DATA (an out-of-range label was flagged by an earlier backward; the flag is
 * checked without synchronising, so it is reported one call late), SMLP_E_CUDA. */
int sparse_mlp_backward(smlp_handle* h, const int32_t* labels, const int32_t* y_idx,
                        float* loss, const smlp_sgd* fused);

/* sparse_mlp_step — Eq. 1 update on the grad view (after the caller's SUM allreduce and
 * with sgd->grad_scale = 1/K).  Errors: SMLP_E_STATE if no unfused backward is pending. */
int sparse_mlp_step(smlp_handle* h, const smlp_sgd* sgd);

/* One fused training step with HOST buffers (pinned for async copies): H2D of
 * x_host [B x n_1] and y_host [B], forward(train) + fused backward, D2H of the loss.
 * The copies are enqueued on the handle's stream; SYNC at the end (loss is ready). */
int sparse_mlp_train_step_host(smlp_handle* h, const float* x_host, const int32_t* y_host,
                               int32_t B, uint64_t step, const smlp_sgd* sgd, float* loss_host);

/* sparse_mlp_train_step_host_async — the same step, pipelined: x_host / y_host go to one of two
 * device staging buffers on an internal copy stream (waiting only for the forward that last
 * read that buffer, two calls ago), so the H2D of step s+1 overlaps the compute of step s.
 * ASYNC: returns once enqueued.  x_host, y_host and loss_host must be PINNED host memory and
 * stay valid / unread until sparse_mlp_sync (loss_host: host float or NULL). */
int sparse_mlp_train_step_host_async(smlp_handle* h, const float* x_host, const int32_t* y_host,
                                     int32_t B, uint64_t step, const smlp_sgd* sgd, float* loss_host);

/* sparse_mlp_sync — SYNC: waits for all work enqueued on the handle's stream; reports a
 * deferred device error (SMLP_E_DATA label out of range). */
int sparse_mlp_sync(smlp_handle* h);

/* sparse_mlp_join — enqueue on the handle's stream the waits for work the library left running
 * on its side stream: the Eq. 1 pass (sparse_mlp_backward with SGD / sparse_mlp_step) refreshes
 * each layer's mirror-ordered weight copy there and joins it lazily (the next forward waits for
 * layer l's copy right before layer l; every other call joins all first).  No host sync; CUDA-
 * graph capturable.  A stream capture that contains a training step must call it before the
 * capture ends (the side-stream work has to rejoin the capturing stream).  Errors: SMLP_E_ARG
 * (NULL handle), SMLP_E_CUDA. */
int sparse_mlp_join(smlp_handle* h);

/* Contiguous device views [values of W^(2..L) at their capacity offsets || biases b_2..b_L],
 * identical layout on every replica, stable for the life of the handle (holes left by
 * pruning are zero).  grad view: filled by an unfused backward (X1 allreduce, SUM).
 * param view: the parameters theta = (w, b) (X2 averaging, Eq. 2). */
int sparse_mlp_grad_view(smlp_handle* h, float** dev, int64_t* count, uint64_t* version);
int sparse_mlp_param_view(smlp_handle* h, float** dev, int64_t* count, uint64_t* version);

/* sparse_mlp_gradient_flow — PAPER.md:315 ("the first-order approximation of the decrease in
 * the loss expected after a gradient step"): the squared L2 norm of the
 * pending gradient of an unfused backward, sum over W^(2..L) of sum g^2 over the existing
 * connections plus sum gb^2 over the biases, accumulated in fp64 in a fixed order
 * (deterministic).  *out_host: host double.  SYNC.  Errors: SMLP_E_STATE if no unfused
 * backward's gradient is pending. */
int sparse_mlp_gradient_flow(smlp_handle* h, double* out_host);

/* sparse_mlp_export_positions — the entries of W^(l) in canonical order as device arrays:
 * pos_dev[k] = i * n_l + j (uint64), val_dev[k] = w_ij; both caller-owned device buffers of at
 * least nnz(W^(l)) elements (sparse_mlp_info).  ASYNC.  Used to all-gather replicas' supports. */
int sparse_mlp_export_positions(smlp_handle* h, int32_t l, uint64_t* pos_dev, float* val_dev);

/* sparse_mlp_union_average_layer — WASAP phase-2 averaging (Alg. 1, Eq. 2
 * PAPER.md:94-96, re-sparsification PAPER.md:97-98) of W^(l) over the
 * UNION of K replicas' supports.  pos_all / val_all: device arrays of `total` entries, the K
 * replicas' sparse_mlp_export_positions lists concatenated in rank order.  Per distinct position:
 * fp32 sum of the present values in rank order, / K in fp32 (absent = 0; DESIGN R31); then the
 * union entries closest to zero are removed (key |w| bits, ties by position) down to `target`
 * connections; the rest become W^(l) with momentum 0.  Deterministic, so replicas that pass the
 * same inputs end bit-identical.  *kept (host, may be NULL) = min(target, union size).
 * version += 1.  SYNC.  Errors: SMLP_E_ARG (l, K < 1, target > capacity), SMLP_E_NOMEM. */
int sparse_mlp_union_average_layer(smlp_handle* h, int32_t l, int32_t K, const uint64_t* pos_all,
                                   const float* val_all, int64_t total, int64_t target, int64_t* kept);

/* sparse_mlp_retain_valid_updates — RetainValidUpdates of Alg. 1 (Fig. 4
 * PAPER.md:81-89): a gradient of W^(l) computed on an
 * older topology (stale_pos: its sorted canonical positions i * n_l + j, stale_g: the gradient
 * values, both device arrays of n_stale entries, e.g. sparse_mlp_export_positions + the grad view
 * slice at that version) is mapped onto the CURRENT support: each current connection takes the
 * stale gradient at its position, or 0 if the connection did not exist then (the intersection of
 * the two supports).  Written into W^(l)'s slice of the grad view; the bias slices are left to the
 * caller; then sparse_mlp_step applies Eq. 1.  *retained (host, may be NULL) = size of the
 * intersection.  Pure data movement (bit-exact).  SYNC. */
int sparse_mlp_retain_valid_updates(smlp_handle* h, int32_t l, const uint64_t* stale_pos,
                                    const float* stale_g, int64_t n_stale, int64_t* retained);

/* sparse_mlp_wait_layer — makes `stream` (a cudaStream_t) wait until the last backward's
 * gradient of W^(l) (and of b_{l-1}) is final, so that layer's slice of the grad view can be
 * allreduced while the backward of the layers below continues (SURVEY §8(e) overlap; the
 * output layer finishes first).  ASYNC.  Errors: SMLP_E_ARG (l not in [2, L]), SMLP_E_STATE
 * (no backward ran yet). */
int sparse_mlp_wait_layer(smlp_handle* h, int32_t l, void* stream);

/* sparse_mlp_view_layout — where each layer lives in the grad / param views: host int64
 * arrays val_off[L-1], cap[L-1] (index l-2 = W^(l), floats) and *bias_base (start of
 * b_2 || ... || b_L, through the end of the view).  Any pointer may be NULL. */
int sparse_mlp_view_layout(smlp_handle* h, int64_t* val_off, int64_t* cap, int64_t* bias_base);

/* Call after writing the param view directly (e.g. the Eq. 2 averaging allreduce): refreshes
 * the forward's mirror-ordered copy of the weights.  Asynchronous, graph-capturable. */
int sparse_mlp_params_updated(smlp_handle* h);

/* sparse_mlp_params_averaged — the division of Eq. 2 (theta = (1/K) sum_k
 * theta_k): after the caller SUM-allreduced the param view over K identical-support replicas
 * (all of it, or only its bias block [bias_base, count) when biases_only != 0), every value is
 * divided by K in fp32 (one rounding of the summed value) and, for the full view, the forward's
 * mirror-ordered weight copy is refreshed.  Momentum stays local (R-O10).  Asynchronous on the
 * handle's stream, graph-capturable.  Errors: SMLP_E_ARG if K < 1.                            */
int sparse_mlp_params_averaged(smlp_handle* h, int32_t K, int32_t biases_only);

/* sparse_mlp_evolve_topology — Alg. 2 PAPER.md:659-664 on every weight layer that is not
 * dense-capped: per sign class k = floor(zeta n_+/-), remove the k positives and the k
 * negatives closest to zero (key: |w| bits, canonical index; R5-R7), regrow R = k_+ + k_-
 * connections at the first R distinct positions of the REGROW Philox stream (counter
 * evolve_idx) that are outside the pre-call support and join two alive neurons (R8); new
 * w from the init scheme, new v = 0; survivors keep (w, v) bit-exactly.  A layer with
 * fewer free positions than R is left unchanged (R9).  Deterministic in (seed, evolve_idx,
 * weights), so replicas agree without communication.  version += 1.
 *   removed_per_layer: host int64 [L] or NULL; index l-1 = removed count of W^(l), -1 =
 *   skipped (dense-capped or saturated).
 * SYNC (small count read-backs).  Errors: SMLP_E_ARG if zeta not in (0, 1). */
int sparse_mlp_evolve_topology(smlp_handle* h, double zeta, uint64_t evolve_idx,
                               int64_t* removed_per_layer);

/* sparse_mlp_prune_neurons — Importance Pruning, Alg. 2 PAPER.md:652-658 with Eq. 4
 * I_j = sum_i |w_ij| (sequential fp64 sum, ascending i) over the hidden
 * layers h = 2..L-1, all importances taken before any removal (R19); threshold
 * t = percentile(alive I, `percentile`) by linear interpolation (R15); alive neurons with
 * I_j < t lose their incoming column of W^(h) and, with SMLP_PRUNE_OUTGOING, their outgoing
 * row of W^(h+1) (R17); a layer that would lose every alive neuron is skipped.  version += 1.
 *   pruned_per_layer: host int64 [L] or NULL (index l-1; -1 = skipped).
 *   removed_conn:     host int64 [L] or NULL (index l-1 = connections removed from W^(l)).
 * SYNC.  Errors: SMLP_E_ARG if percentile not in [0, 100). */
int sparse_mlp_prune_neurons(smlp_handle* h, double percentile, int32_t flags,
                             int64_t* pruned_per_layer, int64_t* removed_conn);

/* Eq. 4 importances of neuron layer l (2..L-1) into out [n_l] (device or host fp64). SYNC. */
int sparse_mlp_importance(smlp_handle* h, int32_t l, double* out, int32_t to_host);

/* Model information (host struct).  SYNC-free (host-side bookkeeping). */
int sparse_mlp_info(smlp_handle* h, smlp_info* info);

/* Export W^(l) (l = 2..L) in the paper orientation: CSR by input row i (row_ptr [n_{l-1}+1],
 * col_idx / val / mom [nnz]) with sorted unique columns.  to_host: 1 = host buffers, 0 =
 * device buffers.  Any pointer may be NULL to skip that array.  SYNC. */
int sparse_mlp_export_layer(smlp_handle* h, int32_t l, int32_t* row_ptr, int32_t* col_idx,
                            float* val, float* mom, int32_t to_host);

/* Import W^(l) from HOST arrays (parity tests / checkpoints).  nnz must not exceed the
 * layer's capacity.  The invariants of SPEC S:26-29 are checked (row_ptr monotone from 0 to
 * nnz, columns sorted unique within rows and in [0, n_l)); on violation SMLP_E_STRUCT names
 * the offending (row, col).  Rebuilds the output-major mirror; version += 1.  SYNC. */
int sparse_mlp_import_layer(smlp_handle* h, int32_t l, int64_t nnz, const int32_t* row_ptr,
                            const int32_t* col_idx, const float* val, const float* mom);

/* Biases b_l / momentum of b_l (l = 2..L) and liveness of neuron layer l (1..L), host. SYNC. */
int sparse_mlp_export_bias(smlp_handle* h, int32_t l, float* bias, float* bias_mom);
int sparse_mlp_import_bias(smlp_handle* h, int32_t l, const float* bias, const float* bias_mom);
int sparse_mlp_export_alive(smlp_handle* h, int32_t l, uint8_t* alive);
int sparse_mlp_import_alive(smlp_handle* h, int32_t l, const uint8_t* alive);

/* Trace export for parity tests: kind 0 = activations a_l (l = 1..L-1; l = L gives the
 * logits z_L), kind 1 = deltas delta_l (l = 2..L) of the last forward / backward, as host
 * fp32 row-major [B x n_l].  kind 2 = gradient of W^(l) values from the grad view (host
 * fp32 [nnz]) and kind 3 = bias gradient of layer l (host fp32 [n_l]).  kind 4 (l ignored):
 * out[0] = 1 if the last forward took the exact binary-input path of W^(2) (every input value
 * 0 or 1), 0 if it took the fp32 gather path, -1 if the path is disabled
 * (padded batch > 128).  SYNC. */
int sparse_mlp_export_trace(smlp_handle* h, int32_t kind, int32_t l, float* out);

/* Per-kernel timing with CUDA events on the handle's stream (bench.py's roofline evidence).
 * sparse_mlp_profile(h, 1) clears the records and starts recording an event pair around every
 * hot-path kernel launch; (h, 0) stops.  Not usable while a CUDA graph is being captured.
 * sparse_mlp_profile_read (SYNC) aggregates the recorded launches by (kind, layer): kind
 * 0 stage_input, 1 fwd, 2 fwd_finish, 3 softmax_ce, 4 bwd, 5 bwd_finish, 6 sgd_update.
 * bytes_per_launch / flops_per_launch are the ALGORITHMIC figures of DESIGN.md (formula F1 split
 * per launch: index/value terms 12 B/nnz forward, 20 B/nnz fused backward (12 unfused), 20 B per
 * value for sgd_update, activation terms 4 B per batch column per neuron read or written). */
typedef struct {
    int32_t kind;
    int32_t layer;
    int64_t launches;
    double  total_ms;
    double  bytes_per_launch;
    double  flops_per_launch;
} smlp_kernel_stat;
int sparse_mlp_profile(smlp_handle* h, int32_t enable);
int sparse_mlp_profile_read(smlp_handle* h, smlp_kernel_stat* out, int32_t cap, int32_t* n);

/* Dropout step source for CUDA-graph replay: when dev_counter is non-NULL, train-mode forward
 * reads the dropout stream counter (R13) from *dev_counter (device uint64) at kernel time
 * instead of its `step` argument, so one captured graph draws fresh masks on every replay
 * (the caller advances the counter, e.g. inside the same graph).  NULL restores `step`. */
int sparse_mlp_set_step_counter(smlp_handle* h, const uint64_t* dev_counter);

/* Last error text of this handle (or of the last failed create when h is NULL). */
const char* sparse_mlp_last_error(const smlp_handle* h);

/* Library version string. */
const char* sparse_mlp_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SPARSE_MLP_H */
