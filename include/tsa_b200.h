/*
 * tsa_b200.h -- C ABI of the B200-native Token Sparse Attention prefill path.
 *
 * This is the drop-in boundary for the reference's operator API
 * (/root/reference/proj/include/tsa/{token_coverage,attention}.hpp): every
 * entry point below replaces one reference function (cited per entry) with a
 * stream-ordered CUDA implementation for sm_100a.  The signatures use only
 * plain pointers, sizes and a POD descriptor -- no torch, no Eigen -- so any
 * FFI (ctypes, cgo, JNI, a C++ adapter: include/tsa_b200.hpp) can bind them.
 *
 * Conventions
 *  - Tensor layout is the reference's HeadTensors (attention.hpp:16-25):
 *    q = H blocks of [L x d] row-major, k/v = Hkv blocks of [L x d];
 *    kv_head(h) = h / (H / Hkv).  Element type per `dtype` (f32 or bf16).
 *  - Scores are f32 [H x L] (HeadScores::s, token_coverage.hpp:12-20).
 *  - Index lists are int32 [H x L] rows, of which the first k_keep entries of
 *    each row are valid and strictly ascending (TokenSelection::indices,
 *    selection.hpp:12-21).  k_keep lives in device memory (int32) so the
 *    chain runs without a host round trip.
 *  - All pointers are device pointers unless named *_host; every call is
 *    asynchronous on `stream` (a cudaStream_t passed as void*; NULL = legacy
 *    default stream).
 *  - Errors: a non-zero return code; tsa_last_error() names the violated
 *    precondition with the reference's wording (std::invalid_argument there).
 *    TSA_ERR_INVALID = precondition, TSA_ERR_CUDA = launch/runtime failure.
 *  - Multi-GPU head sharding: [head_begin, head_end) selects the query heads a
 *    call computes (GQA aligned).  Score rows and outputs of other heads are
 *    left untouched, so the caller exchanges them (all-gather) between calls.
 */
#ifndef TSA_B200_H_
#define TSA_B200_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define TSA_API __attribute__((visibility("default")))
#else
#define TSA_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

enum tsa_dtype { TSA_F32 = 0, TSA_BF16 = 1 };
/* SparseMode, model.hpp:51 */
enum tsa_mode { TSA_MODE_DENSE = 0, TSA_MODE_DYNAMIC = 1, TSA_MODE_FIXED = 2 };
/* ForcedPolicy, model.hpp:54 */
enum tsa_forced_policy { TSA_FORCED_FINAL_TOKEN = 0, TSA_FORCED_RECENT_WINDOW = 1 };
enum tsa_status { TSA_OK = 0, TSA_ERR_INVALID = 1, TSA_ERR_CUDA = 2, TSA_ERR_NCCL = 3 };
/* Scoring arithmetic: REFERENCE reproduces the reference's f32 operation
 * order bit for bit (sequential-order logits, glibc's expf, sequential softmax
 * sums; bf16 d = 128 runs the fused kernels of score_exact.cu); FAST runs
 * Q K^T on the tensor cores with approximate exponentials (bf16 only; scores
 * within ~1e-5 relative, so k_keep / index sets may differ at near ties).
 * DEFAULT = REFERENCE. */
enum tsa_scoring { TSA_SCORING_DEFAULT = 0, TSA_SCORING_REFERENCE = 1, TSA_SCORING_FAST = 2 };

/* One attention layer's geometry plus the SparsePlan parameters
 * (model.hpp:58-73).  Defaults via tsa_desc_init(). */
typedef struct tsa_desc {
    int32_t n_heads;       /* H */
    int32_t n_kv_heads;    /* Hkv, H % Hkv == 0 */
    int32_t seq_len;       /* L */
    int32_t d_head;        /* d in [1, 256] (bf16: even); tensor-core path: bf16, d = 128 */
    int32_t dtype;         /* tsa_dtype */
    int32_t mode;          /* tsa_mode */
    double tau;            /* dynamic coverage, [0, 1]     (SparsePlan::tau = 0.005) */
    double s_fixed;        /* fixed sparsity ratio, [0, 1) (SparsePlan::s_fixed = 0) */
    int32_t last_q;        /* >= 1 (SparsePlan::last_q = 64) */
    int32_t kernel;        /* odd >= 1 (SparsePlan::kernel = 7) */
    int32_t forced_policy; /* tsa_forced_policy (SparsePlan::forced) */
    int32_t head_begin;    /* query-head shard [head_begin, head_end) */
    int32_t head_end;
    int32_t scoring;       /* tsa_scoring */
} tsa_desc;

TSA_API void tsa_desc_init(tsa_desc* d, int32_t n_heads, int32_t n_kv_heads, int32_t seq_len,
                   int32_t d_head, int32_t dtype);
TSA_API const char* tsa_last_error(void);
TSA_API const char* tsa_version(void);
/* Number of kernels this library has launched in the process (all streams). */
TSA_API uint64_t tsa_kernel_launches(void);
/* Destroys the CUDA graphs tsa_sparse_attention_layer keeps (one per
 * descriptor + buffer addresses, at most 16).  Call before freeing buffers a
 * later allocation could reuse with a different meaning. */
TSA_API void tsa_release_graphs(void);

/* Bytes of scratch the calls below need for `d` (scores, index lists,
 * compressed Q/K/V/O buffers and selection scratch), 256-B aligned.
 * tsa_budget, tsa_aggregate_scores and tsa_coverage_budget only touch the
 * first 512 + align256(4 L) bytes. */
TSA_API int tsa_workspace_size(const tsa_desc* d, size_t* bytes);

/* --- the path, stage by stage ------------------------------------------ */

/* score_tokens (token_coverage.hpp:32 / token_coverage.cpp:16-50).
 * Writes s[h, :] for h in the shard; s is [H x L] f32. */
TSA_API int tsa_score(const tsa_desc* d, const void* q, const void* k, float* s, void* ws, void* stream);

/* The softmax exponential of REFERENCE scoring, elementwise on the device:
 * y[i] = expf(x[i]) exactly as glibc computes it (std::exp(float),
 * tensor_ops.cpp:62), for x <= 0.  Exported so the parity suite can pin the
 * port against the host libm. */
TSA_API int tsa_expf(const float* x, float* y, int64_t n, void* stream);

/* aggregate_scores + coverage_budget (token_coverage.cpp:52-96) for
 * TSA_MODE_DYNAMIC, fixed_budget (:98-109) for TSA_MODE_FIXED, L for
 * TSA_MODE_DENSE; min_keep = max(1, |forced|) (model.cpp:172).  Reads all H
 * score rows.  Writes *k_keep (device int32). */
TSA_API int tsa_budget(const tsa_desc* d, const float* s, int32_t* k_keep, void* ws, void* stream);

/* aggregate_scores alone (token_coverage.cpp:52-66): sl[t] = sum_h s[h, t] /
 * total, f32, same operation order as the reference.  Reads all H rows. */
TSA_API int tsa_aggregate_scores(const tsa_desc* d, const float* s, float* sl, void* ws,
                                 void* stream);

/* coverage_budget alone (token_coverage.cpp:68-96) on a LayerScores vector
 * sl [L] with the descriptor's tau and an explicit min_keep. */
TSA_API int tsa_coverage_budget(const tsa_desc* d, const float* sl, int32_t min_keep,
                                int32_t* k_keep, void* ws, void* stream);

/* select_tokens (token_coverage.cpp:111-152) for the shard's heads with an
 * explicit forced list (device int32, sorted, unique, in range -- the host
 * adapter normalises it as the reference does at :113-121).  idx rows are
 * [L] wide; inv (optional, may be NULL) receives the inverse map
 * inv[h, t] = position of t in idx[h] or -1. */
TSA_API int tsa_select(const tsa_desc* d, const float* s, const int32_t* k_keep, const int32_t* forced,
               int32_t n_forced, int32_t* idx, int32_t* inv, void* ws, void* stream);

/* gather_rows x3 (tensor_ops.cpp:92-99 via attention.cpp:93-95): qc/kc/vc
 * are [H x L x d] with the first k_keep rows of each head valid (K/V rows
 * come from the head's KV group, duplicated per query head).  qc may be NULL
 * (K/V only, for tsa_attend_indexed). */
TSA_API int tsa_gather(const tsa_desc* d, const void* q, const void* k, const void* v,
               const int32_t* idx, const int32_t* k_keep, void* qc, void* kc, void* vc,
               void* stream);

/* The `inner` seam (AttentionKernel, attention.hpp:28) with its default
 * dense_causal_attention (attention.cpp:25-40): causal attention over the
 * first n rows of each head, n = *k_keep (device).  kv_group = 1 when K/V
 * are per query head (compressed), H/Hkv when they are the KV heads. */
TSA_API int tsa_attend(const tsa_desc* d, const void* qc, const void* kc, const void* vc,
               const int32_t* k_keep, int32_t kv_group, void* oc, void* stream);

/* scatter_rows (tensor_ops.cpp:101-112 via attention.cpp:96): out[h, t] =
 * oc[h, inv[h, t]] or +0.0 (every row of the shard written once). */
TSA_API int tsa_scatter(const tsa_desc* d, const void* oc, const int32_t* inv, void* out, void* stream);

/* Fused attend + decompress for bf16 / d = 128 (the production path of
 * tsa_sparse_attention_layer): Q rows are fetched from the original q by idx
 * with TMA gather4, K/V tiles from the compressed per-head kc/vc
 * (tsa_gather_zero), causal attention runs over the first k_keep rows, and each
 * output row is stored at its original position out[h, idx[h, r]].  When
 * k_keep == L the selection is the identity and the K/V tiles are read in
 * place from k / v (the KV heads; kc / vc are not read).  Rows not selected are
 * left untouched -- pair with tsa_gather_zero or tsa_zero_unselected. */
TSA_API int tsa_attend_indexed(const tsa_desc* d, const void* q, const void* k, const void* v,
                               const void* kc, const void* vc, const int32_t* idx,
                               const int32_t* k_keep, void* out, void* stream);

/* K/V half of tsa_gather (kc, vc) and tsa_zero_unselected in one pass: the
 * two independent HBM streams of the fused path share a launch.  When
 * k_keep == L the copy is skipped (tsa_attend_indexed reads K/V in place). */
TSA_API int tsa_gather_zero(const tsa_desc* d, const void* k, const void* v, const int32_t* idx,
                            const int32_t* k_keep, void* kc, void* vc, const int32_t* inv,
                            void* out, void* stream);

/* --- the multi-GPU exchanges fused into the producers (peer memory) ---
 * The budget sums the score rows of every head (token_coverage.cpp:55-57) and
 * the head concat before W_O (model.cpp:197-200) needs every head's output on
 * every rank.  Instead of all-gathers between the kernels, the kernels that
 * write score rows (the pool pass of tsa_score) and output rows (the zero rows
 * and the attention epilogue) store each row of the shard's heads to all
 * n_outs bases: row t of the descriptor's head h (head_begin <= h < head_end)
 * lands at outs[i] + (h L + t) d in each -- outs[i] is the base of an
 * [H x L x d] buffer, this rank's and each peer's mapped into this device's
 * address space over NVLink (CUDA IPC: tsa_ipc_alloc / tsa_ipc_open below),
 * offset by h0 L d when the descriptor numbers a shard's heads from 0 (as
 * dist.py's per-rank descriptors do).  The kernels end with a
 * system-scope fence; the caller orders the peers' reads after them with a
 * cross-rank barrier on the stream.  1 <= n_outs <= TSA_MAX_REPLICAS. */
#define TSA_MAX_REPLICAS 8
/* tsa_score with each score row written to every replica: row h of the
 * descriptor's heads lands at s_outs[i] + h * L (f32) -- the score all-gather
 * before the budget. */
TSA_API int tsa_score_replicas(const tsa_desc* d, const void* q, const void* k,
                               float* const* s_outs, int32_t n_outs, void* ws, void* stream);
TSA_API int tsa_gather_zero_replicas(const tsa_desc* d, const void* k, const void* v,
                                     const int32_t* idx, const int32_t* k_keep, void* kc,
                                     void* vc, const int32_t* inv, void* const* outs,
                                     int32_t n_outs, void* stream);
TSA_API int tsa_attend_indexed_replicas(const tsa_desc* d, const void* q, const void* k,
                                        const void* v, const void* kc, const void* vc,
                                        const int32_t* idx, const int32_t* k_keep,
                                        void* const* outs, int32_t n_outs, void* stream);

/* Peer memory for those exchanges (CUDA IPC): tsa_ipc_alloc returns a zeroed
 * device buffer and its 64-byte handle, which the other ranks map with
 * tsa_ipc_open (over NVLink between GPUs; ranks sharing a device work too).
 * tsa_peer_barrier is a cross-rank barrier on the stream over one channel's
 * signal arrays: signals[r] is rank r's int32 [world + 2] array (this rank's
 * own and the mapped peers'; zeroed before first use): slots [0, world) take
 * the arrivals, [world] is the rank's epoch counter, [world + 1] a timeout
 * flag.  With epoch < 1 the epoch is the device counter + 1 (graph-capturable:
 * every rank runs the same barrier sequence); epoch >= 1 uses the host's value.
 * The call stores the epoch into slot [rank] of every array (system-scope
 * release, after a system fence) and waits until this rank's array holds >=
 * epoch in every slot (acquire).  A peer that has not arrived within
 * TSA_PEER_TIMEOUT_S seconds (environment, default 600 -- NCCL's) sets the
 * timeout flag and the barrier returns instead of trapping; tsa_peer_check
 * reads the flags of this rank's n_channels consecutive arrays (synchronous)
 * and fails with TSA_ERR_CUDA if one is set. */
#define TSA_IPC_HANDLE_BYTES 64
TSA_API int tsa_ipc_alloc(size_t bytes, void** ptr, void* handle);
TSA_API int tsa_ipc_open(const void* handle, void** ptr);
TSA_API int tsa_ipc_close(void* ptr);
TSA_API int tsa_ipc_free(void* ptr);
TSA_API int tsa_peer_barrier(int32_t* const* signals, int32_t world, int32_t rank, int32_t epoch,
                             void* stream);
TSA_API int tsa_peer_check(const int32_t* own_signals, int32_t world, int32_t n_channels,
                           void* stream);

/* The head-sharded layer in one call (model.cpp:169-183 with the heads of the
 * layer split over world ranks, one process per GPU).  d holds
 * the WHOLE layer's geometry with [head_begin, head_end) = this rank's shard
 * (whole KV groups); q / k / v are this rank's heads ([head_end - head_begin,
 * L, d] and their KV heads).  ws: tsa_workspace_size(d) bytes.  k_keep
 * (device int32) is the layer's budget (identical on every rank).  Exactly
 * one exchange form:
 *  - peer (tsa_peer, CUDA IPC buffers every rank allocated and mapped): the
 *    score rows go from the pool pass straight into every rank's [H x L]
 *    buffer, the output rows from the zero-row pass and the attention
 *    epilogue into every rank's [H x L x d] buffer (out[rank] holds the
 *    gathered layer output when the call completes on the stream); device
 *    barriers on signals[0..2] order the step (graph-capturable; bf16, d 128);
 *  - nccl_comm (an ncclComm_t over the same ranks, rank = shard index): the
 *    score rows are all-gathered in place in s_full [H x L] before the budget
 *    and the outputs in out_full [H x L x d] after the attention
 *    (ncclAllGather, libnccl.so.2 resolved at run time).
 * TSA_MODE_DENSE runs the dense kernel on the shard and the same output
 * exchange. */
typedef struct tsa_peer {
    int32_t world, rank;
    float* scores[TSA_MAX_REPLICAS];            /* every rank's [H x L] f32 buffer, rank order */
    void* out[TSA_MAX_REPLICAS];                /* every rank's [H x L x d] buffer */
    int32_t* signals[3][TSA_MAX_REPLICAS];      /* per channel: every rank's int32 [world + 2] */
} tsa_peer;
TSA_API int tsa_sparse_attention_layer_sharded(const tsa_desc* d, const void* q, const void* k,
                                               const void* v, const tsa_peer* peer,
                                               void* nccl_comm, float* s_full, void* out_full,
                                               int32_t* k_keep, void* ws, void* stream);

/* out[h, t] = +0.0 for every t with inv[h, t] < 0 (scatter_rows' zero rows). */
TSA_API int tsa_zero_unselected(const tsa_desc* d, const int32_t* inv, void* out, void* stream);

/* scatter_rows for a caller-supplied selection: builds the inverse map of
 * idx (first k_keep entries per head) in ws, then tsa_scatter. */
TSA_API int tsa_scatter_rows(const tsa_desc* d, const void* oc, const int32_t* idx,
                             const int32_t* k_keep, void* out, void* ws, void* stream);

/* Synchronises `stream` and reports device-side precondition failures
 * recorded in ws by tsa_budget (aggregate_scores on all-zero scores,
 * token_coverage.cpp:62-64), then clears them. */
TSA_API int tsa_check(const tsa_desc* d, void* ws, void* stream);

/* --- composite calls ---------------------------------------------------- */

/* token_sparse_attention (attention.hpp:44-45) given a selection. */
TSA_API int tsa_token_sparse_attention(const tsa_desc* d, const void* q, const void* k, const void* v,
                               const int32_t* idx, const int32_t* k_keep, void* out, void* ws,
                               void* stream);

/* Dense causal attention of every head directly on q/k/v (the tau = 0 /
 * dense-layer branch, model.cpp:184-194): the baseline the sparse path is
 * measured against. */
TSA_API int tsa_dense_attention(const tsa_desc* d, const void* q, const void* k, const void* v, void* out,
                        void* stream);

/* The sparse-layer branch of layer_forward (model.cpp:169-183) on one GPU:
 * score -> budget -> select -> gather -> attend -> scatter.  idx_out
 * (optional) receives the selection [H x L] int32, k_keep_out (device int32,
 * required) the budget; k_keep_host (optional, pinned) is filled
 * asynchronously for LayerStat.  Multi-GPU callers use the stage entry points
 * with an all-gather of s between tsa_score and tsa_budget.
 * The chain never waits on the host, so its launches are captured into a CUDA
 * graph on the first call for a (descriptor, buffer addresses) key and
 * replayed afterwards (TSA_GRAPHS=0 disables; calls on a capturing stream run
 * eagerly into the caller's capture). */
TSA_API int tsa_sparse_attention_layer(const tsa_desc* d, const void* q, const void* k, const void* v,
                               void* out, int32_t* idx_out, int32_t* k_keep_out,
                               int32_t* k_keep_host, void* ws, void* stream);

/* The layer on HOST tensors (the reference's calling convention: its operators
 * take host matrices): q/k/v/out_host [H|Hkv][L][d] in host memory (pinned for
 * asynchronous copies), q/k/v/out device staging buffers of the same shapes.
 * The transfers are pipelined with the compute: the Q tail rows first, then K
 * two KV heads at a time, each pair scored as soon as it has arrived (scoring
 * needs all of K before the budget, so all but the last pair's scoring hides
 * under the copy); then, per group of n_groups (0 = one per KV head), the
 * group's V heads and its Q rows head by head: the group's K/V are compressed
 * once, each head's attention starts when its Q rows have arrived and its
 * output rows are copied back while the next head computes (more than 64 query
 * heads: whole groups, the first and last head by head).  Completion on
 * `stream` covers every copy; a caller may overlap consecutive calls by
 * alternating two buffer sets (q..out, ws) on two streams.  f32 / d != 128 /
 * dense mode: one copy in, the layer, one copy out. */
TSA_API int tsa_sparse_attention_layer_host(const tsa_desc* d, const void* q_host,
                                            const void* k_host, const void* v_host,
                                            void* out_host, void* q, void* k, void* v, void* out,
                                            int32_t* idx_out, int32_t* k_keep_out,
                                            int32_t* k_keep_host, void* ws, int32_t n_groups,
                                            void* stream);

/* ---- Attention-branch producer / consumer (layer_forward, model.cpp:169-201) ----
 * The unfused stages around the path: rms_norm, RoPE + head split, head
 * concat (a caller's BLAS does the projections between them); the fused
 * tcgen05 projections that replace the whole chain follow below
 * (tsa_qkv_proj, tsa_out_proj_residual).  Row-major, dtype TSA_F32 or
 * TSA_BF16 (compute in f32). */

/* rms_norm (model.cpp:81-94): out[r] = (x[r] * inv_r) * gain, inv_r =
 * 1 / sqrt(sum_j x[r, j]^2 / cols + eps), the sum taken sequentially in f32 as
 * the reference does (f32 inputs match it bit for bit). */
TSA_API int tsa_rms_norm(const void* x, const float* gain, int64_t rows, int32_t cols, float eps,
                         int32_t dtype, void* out, void* stream);

/* RoPE angles of apply_rope (model.cpp:107-116) at positions 0..seq_len-1:
 * table[t][i] = {(float)cos(t w_i), (float)sin(t w_i)}, w_i = theta^(-2i/d)
 * (double, host libm), f32 [seq_len][d_head/2][2]. */
TSA_API int tsa_rope_table(int32_t seq_len, int32_t d_head, float theta, float* table,
                           void* stream);

/* split_heads + apply_rope of project_qkv (model.cpp:128-158): projection rows
 * qkv [L][(H + 2 Hkv) d] (q heads, then k heads, then v heads) -> q [H][L][d],
 * k / v [Hkv][L][d]; q and k rotated in f32 (x0 c - x1 s, x0 s + x1 c). */
TSA_API int tsa_split_heads_rope(const tsa_desc* d, const void* qkv, const float* table, void* q,
                                 void* k, void* v, void* stream);

/* Head concat before W_o (model.cpp:196-200): heads [H][L][d] -> cat [L][H d]. */
TSA_API int tsa_heads_concat(const tsa_desc* d, const void* heads, void* cat, void* stream);

/* ---- The projections on the tensor cores, with the work around them fused ----
 * Hand-written tcgen05 GEMMs (bf16 in, f32 accumulation in TMEM): one
 * persistent kernel per projection, 128 x 256 tiles.  These replace the
 * caller's BLAS calls of project_qkv (model.cpp:139-158) and the W_O
 * projection (model.cpp:196-201) and absorb the passes around them. */

/* c [M][N] = a [M][K] * b_t [N][K]^T (bf16, N % 256 == 0, K % 64 == 0). */
TSA_API int tsa_gemm_bf16(const void* a, const void* b_t, void* c, int32_t M, int32_t N, int32_t K,
                          void* stream);

/* Weight layout for the projections, done once per weight: w_t [cols][rows]
 * bf16 = (diag(gain) w)^T for w [rows][cols] (dtype TSA_F32 / TSA_BF16).  For
 * W_qkv pass the attention-norm gain (rms_norm's gain folds into the weight);
 * for W_o pass gain = NULL. */
TSA_API int tsa_prepare_weight(const void* w, int32_t dtype, const float* gain, int32_t rows,
                               int32_t cols, void* w_t, void* stream);

/* inv[r] = 1 / sqrt(sum_j x[r, j]^2 / cols + eps) for bf16 x [rows][cols]
 * (rms_norm's row statistic, model.cpp:81-94; cols % 8 == 0). */
TSA_API int tsa_row_inv_rms(const void* x, int64_t rows, int32_t cols, float eps, float* inv,
                            void* stream);

/* project_qkv (model.cpp:128-158) with rms_norm (model.cpp:81-94) folded in,
 * one GEMM: q [H][L][d], k / v [Hkv][L][d] = split_heads(rope(
 * (inv_rms[t] * x[t]) W')) for x [L][d_model] bf16 and w_t from
 * tsa_prepare_weight(W_qkv, gain) ([(H + 2 Hkv) d][d_model]); inv_rms from
 * tsa_row_inv_rms (NULL: no norm); table from tsa_rope_table.  RoPE rotates in
 * f32 (x0 c - x1 s, x0 s + x1 c) before the single bf16 rounding.  bf16,
 * d_head 128, d_model % 64 == 0, (H + 2 Hkv) d % 256 == 0. */
TSA_API int tsa_qkv_proj(const tsa_desc* d, const void* x, int32_t d_model, const void* w_t,
                         const float* inv_rms, const float* table, void* q, void* k, void* v,
                         void* stream);

/* The W_O projection and residual (model.cpp:196-201): x [L][d_model] +=
 * concat_h(o_h) W_o, reading o [H][L][d] directly (no concat buffer); wo_t =
 * tsa_prepare_weight(W_o, NULL) ([d_model][H d]).  bf16, d_head 128,
 * d_model % 256 == 0.  The sum is rounded to bf16 once. */
TSA_API int tsa_out_proj_residual(const tsa_desc* d, const void* o, const void* wo_t,
                                  int32_t d_model, void* x, void* stream);

/* ---- Drift calibration (drift.hpp, drift.cpp:14-65) ----
 * compute_drift for one layer boundary: *r_out (device double) = mean over
 * the rows t of |next[t] - prev[t]|_2 / (|prev[t]|_2 + epsilon), with the
 * sums in double in the reference's order (j, then t ascending; f32 inputs
 * match it bit for bit).  ws: rows doubles of device scratch. */
TSA_API int tsa_layer_drift(const void* prev, const void* next, int64_t rows, int32_t cols,
                            int32_t dtype, double epsilon, double* r_out, void* ws, void* stream);

/* select_sparse_layers (host): R_hat[l] = #{k : R[k] <= R[l]} / n and the
 * layers with R_hat <= delta, ascending (layers needs room for n). */
TSA_API int tsa_select_sparse_layers(const double* R, int32_t n, double delta, double* R_hat,
                                     int32_t* layers, int32_t* n_layers);

#ifdef __cplusplus
}
#endif
#endif /* TSA_B200_H_ */
