// Shared host/device definitions for the TSA B200 kernels.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <array>
#include <cstdint>
#include <functional>
#include <string>

#include "../../include/tsa_b200.h"

namespace tsa {

constexpr int kNumSMs = 148;  // B200; grids that must fill the GPU use num_sms()

// SM count of the current device (queried once per device).
int num_sms();
// cudaFuncAttributeMaxDynamicSharedMemorySize for `fn` on the current device,
// set once per (device, kernel) -- the attribute is per device context -- and
// thread safe.
int ensure_smem_attr(const void* fn, int bytes);

// Output replicas of the fused multi-GPU boundary: the same [H, L, d] layout
// at up to TSA_MAX_REPLICAS bases (this rank's buffer and the peers'
// symmetric buffers mapped over NVLink).  Kernels write every output row of
// their shard to each base, so the head all-gather (model.cpp:197-200) costs
// no separate pass.  n = 1 is the single-GPU case.
struct OutReplicas {
    void* p[TSA_MAX_REPLICAS];
    int n;
};
inline OutReplicas single_replica(void* p) {
    OutReplicas r{};
    r.p[0] = p;
    r.n = 1;
    return r;
}

// Error state (thread-local, read through tsa_last_error()).
void set_error(const std::string& msg);
int invalid(const std::string& msg);
int cuda_check(cudaError_t e, const char* what);

void count_launch();
void add_launches(unsigned long long n);
unsigned long long launches_so_far();

// graph.cu: capture-once / replay of a launch sequence keyed by the
// descriptor and the buffer addresses it touches.
constexpr int kGraphPtrs = 8;
int graph_launch(const tsa_desc& d, const std::array<const void*, kGraphPtrs>& ptrs,
                 cudaStream_t st, const std::function<int(cudaStream_t)>& body);
void graph_cache_clear();

#define TSA_LAUNCH_CHECK(what)                                             \
    do {                                                                   \
        cudaError_t e_ = cudaGetLastError();                               \
        if (e_ != cudaSuccess) return ::tsa::cuda_check(e_, what);         \
        ::tsa::count_launch();                                             \
    } while (0)

// Element access for the two supported element types.
template <typename T>
struct Elem;
template <>
struct Elem<float> {
    static __device__ __forceinline__ float to_f32(float x) { return x; }
    static __device__ __forceinline__ float from_f32(float x) { return x; }
};
template <>
struct Elem<__nv_bfloat16> {
    static __device__ __forceinline__ float to_f32(__nv_bfloat16 x) { return __bfloat162float(x); }
    static __device__ __forceinline__ __nv_bfloat16 from_f32(float x) { return __float2bfloat16(x); }
};

inline size_t elem_bytes(int dtype) { return dtype == TSA_BF16 ? 2 : 4; }

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Workspace layout (all offsets 256-B aligned).  Sized for the whole layer so
// one allocation serves every stage.
struct Workspace {
    // selection / budget scratch
    size_t status;    // int32 device status word (0 ok, else error code)
    size_t k_keep;    // int32 scratch k_keep for composite calls
    size_t headsum;   // f32 [L]        sum_h s[h, t]
    size_t logits;    // f32 [H x lq x Lp] reference-order logits (REFERENCE / EXACT mode)
    size_t rowstat;   // float2 row partials of FAST scoring (score_fast_rowstat_bytes)
    size_t rowmax;    // int32 [H x lq]  EXACT scoring: encoded row maxima
    size_t rowsum;    // f32 [H x lq]    EXACT scoring: sequential row sums
    size_t colraw;    // f32 [H x L]     raw column sums before the pool
    size_t scores;    // f32 [H x L]
    size_t forced;    // int32 [max(L, 1)]
    size_t idx;       // int32 [H x L]
    size_t inv;       // int32 [H x L]
    size_t qc, kc, vc, oc;  // dtype [H x L x d]
    size_t total;
};

Workspace workspace_layout(const tsa_desc& d);

inline int lq_of(const tsa_desc& d) { return d.last_q < d.seq_len ? d.last_q : d.seq_len; }

bool score_fast_available();
bool score_fast_supported(const tsa_desc& d);
size_t score_fast_rowstat_bytes(const tsa_desc& d);
bool score_exact_supported(const tsa_desc& d);
size_t exact_logits_stride(int L);

// DEFAULT is the reference's arithmetic (bit-exact scores, hence the
// reference's k_keep and index sets); FAST only on request.
inline int scoring_mode(const tsa_desc& d) {
    return d.scoring == TSA_SCORING_DEFAULT ? TSA_SCORING_REFERENCE : d.scoring;
}

// --------------------------------------------------------------- launchers
// score.cu
// s: the [H x L] score rows, or several replicas of them (multi-GPU, each
// rank's buffer); rows of the descriptor's heads are written to every one.
int launch_score_reference(const tsa_desc& d, const void* q, const void* k, const OutReplicas& s,
                           float* logits, int* rowmax, float* rowsum, float* colraw,
                           cudaStream_t st);
// score_exact.cu: the exact row sums, column sums and pool over logits X
// [local head x lq rows, row stride exact_logits_stride(L)] with their
// encoded row maxima (the second half of the exact scorer; REFERENCE-order
// logits of other shapes feed it too)
int launch_score_exact_rows(const tsa_desc& d, float* X, int* rowmax, float* rowsum, float* colraw,
                            const OutReplicas& s, cudaStream_t st);
int launch_fill_int(int* p, int v, int n, cudaStream_t st);
// ordered int encoding of a float (atomicMax of floats as ints)
__device__ __forceinline__ int enc_max(float f) {
    const int i = __float_as_int(f);
    return i >= 0 ? i : i ^ 0x7fffffff;
}
__device__ __forceinline__ float dec_max(int i) { return __int_as_float(i >= 0 ? i : i ^ 0x7fffffff); }
int launch_score_fast(const tsa_desc& d, const void* q, const void* k, const OutReplicas& s,
                      float* logits, float* rowstat, cudaStream_t st);
int launch_expf(const float* x, float* y, int64_t n, cudaStream_t st);
int launch_score_exact(const tsa_desc& d, const void* q, const void* k, const OutReplicas& s,
                       float* X, int* rowmax, float* rowsum, float* colraw, cudaStream_t st);
// select.cu
int launch_budget(const tsa_desc& d, const float* s, int32_t* k_keep, float* headsum,
                  int32_t* status, int min_keep, cudaStream_t st);
int launch_select(const tsa_desc& d, const float* s, const int32_t* k_keep, const int32_t* forced,
                  int32_t n_forced, int32_t forced_begin, int32_t* idx, int32_t* inv,
                  cudaStream_t st);
int launch_aggregate(const tsa_desc& d, const float* s, float* sl, float* headsum,
                     int32_t* status, cudaStream_t st);
int launch_coverage_from_sl(const tsa_desc& d, const float* sl, int32_t* k_keep, int32_t* status,
                            int min_keep, cudaStream_t st);
int launch_write_int(int32_t* dst, int32_t value, cudaStream_t st);
// gather_scatter.cu
int launch_gather(const tsa_desc& d, const void* q, const void* k, const void* v,
                  const int32_t* idx, const int32_t* k_keep, void* qc, void* kc, void* vc,
                  cudaStream_t st);
int launch_gather_zero(const tsa_desc& d, const void* q, const void* k, const void* v,
                       const int32_t* idx, const int32_t* k_keep, void* qc, void* kc, void* vc,
                       const int32_t* inv, void* out, cudaStream_t st);
int launch_scatter(const tsa_desc& d, const void* oc, const int32_t* inv, void* out,
                   cudaStream_t st);
int launch_inverse(const tsa_desc& d, const int32_t* idx, const int32_t* k_keep, int32_t* inv,
                   cudaStream_t st);
int launch_gather_zero_rep(const tsa_desc& d, const void* k, const void* v, const int32_t* idx,
                           const int32_t* k_keep, void* kc, void* vc, const int32_t* inv,
                           const OutReplicas& out, cudaStream_t st);
int launch_zero_unselected(const tsa_desc& d, const int32_t* inv, void* out, cudaStream_t st);
// k / v: the KV heads, read in place when k_keep == L (the identity selection,
// for which launch_gather_zero skips the compressed copy); kc / vc otherwise.
int launch_attend_indexed(const tsa_desc& d, const void* q, const void* k, const void* v,
                          const void* kc, const void* vc, const int32_t* idx,
                          const int32_t* k_keep, void* out, cudaStream_t st);
int launch_attend_indexed_rep(const tsa_desc& d, const void* q, const void* k, const void* v,
                              const void* kc, const void* vc, const int32_t* idx,
                              const int32_t* k_keep, const OutReplicas& out, cudaStream_t st);
int launch_colsum_pool(const tsa_desc& d, const float* probs, const OutReplicas& s,
                       cudaStream_t st);
// producer.cu (attention-branch producer / consumer, model.cpp:81-158, 196-200)
int launch_rms_norm(const void* x, const float* gain, int64_t rows, int cols, float eps, int dtype,
                    void* out, cudaStream_t st);
int launch_rope_table(int seq_len, int d_head, float theta, float* table, cudaStream_t st);
int launch_split_heads_rope(const tsa_desc& d, const void* qkv, const float* table, void* q,
                            void* k, void* v, cudaStream_t st);
int launch_heads_concat(const tsa_desc& d, const void* heads, void* cat, cudaStream_t st);
// proj_gemm.cu: the projections on the tensor cores with fused epilogues
int launch_gemm_bf16(const void* a, const void* b_t, void* c, int M, int N, int K, cudaStream_t st);
int launch_qkv_proj(const tsa_desc& d, const void* x, int d_model, const void* w_t,
                    const float* inv_rms, const float* table, void* q, void* k, void* v,
                    cudaStream_t st);
int launch_out_proj_residual(const tsa_desc& d, const void* o, const void* wo_t, int d_model,
                             void* x, cudaStream_t st);
int launch_row_inv_rms(const void* x, int64_t rows, int cols, float eps, float* inv, cudaStream_t st);
int launch_prepare_weight(const void* w, int dtype, const float* gain, int rows, int cols, void* w_t,
                          cudaStream_t st);
int launch_layer_drift(const void* prev, const void* next, int64_t rows, int cols, int dtype,
                       double eps, double* out, double* ratio_ws, cudaStream_t st);
// attend_simt.cu / attend_sm100.cu
int launch_attend_simt(const tsa_desc& d, const void* q, const void* k, const void* v,
                       const int32_t* n_dev, int32_t n_const, int32_t kv_group, int32_t rows_per_head,
                       int32_t kv_rows_per_head, void* o, cudaStream_t st);
int launch_attend_sm100(const tsa_desc& d, const void* q, const void* k, const void* v,
                        const int32_t* n_dev, int32_t n_const, int32_t kv_group,
                        int32_t rows_per_head, int32_t kv_rows_per_head, void* o,
                        cudaStream_t st);
bool attend_sm100_supported(const tsa_desc& d);
// attend_tf32.cu: f32, d = 128 on the tensor cores (3xTF32)
bool attend_tf32_supported(const tsa_desc& d);
int launch_attend_tf32(const tsa_desc& d, const void* q, const void* k, const void* v,
                       const int32_t* n_dev, int32_t n_const, int32_t kv_group,
                       int32_t rows_per_head, int32_t kv_rows_per_head, void* o, cudaStream_t st,
                       const int32_t* o_rows = nullptr);  // o_rows: scatter row r to o_rows[h, r]
int launch_attend_sm100_rep(const tsa_desc& d, const void* q, const void* k, const void* v,
                            const OutReplicas& o, cudaStream_t st);
// capi.cu (shared with sharded.cu)
int score_stage(const tsa_desc& d, const void* q, const void* k, const OutReplicas& s, void* ws,
                cudaStream_t st);
int budget_stage(const tsa_desc& d, const float* s, int32_t* k_keep, void* ws, int min_keep,
                 cudaStream_t st);
int forced_begin_of(const tsa_desc& d);
int check_descriptor(const tsa_desc* d);
// peer.cu
int launch_peer_barrier(int32_t* const* signals, int world, int rank, cudaStream_t st);

}  // namespace tsa
