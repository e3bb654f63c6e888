// C ABI (include/tsa_b200.h): host-side validation with the reference's
// error wording, workspace layout, and the stage orchestration of the sparse
// layer branch (model.cpp:169-183).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <mutex>
#include <map>
#include <string>
#include <utility>

#include "common.cuh"

namespace tsa {

static thread_local std::string g_error;
static std::atomic<unsigned long long> g_launches{0};

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
void add_launches(unsigned long long n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
unsigned long long launches_so_far() { return g_launches.load(); }

void set_error(const std::string& msg) { g_error = msg; }

int invalid(const std::string& msg) {
    set_error(msg);
    return TSA_ERR_INVALID;
}

int cuda_check(cudaError_t e, const char* what) {
    set_error(std::string(what) + ": " + cudaGetErrorString(e));
    return TSA_ERR_CUDA;
}

int num_sms() {
    static std::atomic<int> cache[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) return kNumSMs;
    if (dev < 64) {
        const int c = cache[dev].load(std::memory_order_relaxed);
        if (c > 0) return c;
    }
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n < 1)
        n = kNumSMs;
    if (dev < 64) cache[dev].store(n, std::memory_order_relaxed);
    return n;
}

int ensure_smem_attr(const void* fn, int bytes) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, int> set_to;  // largest value set so far
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_check(e, "cudaGetDevice");
    std::lock_guard<std::mutex> lock(mu);
    auto it = set_to.find({dev, fn});
    if (it != set_to.end() && it->second >= bytes) return 0;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess) return cuda_check(e, "cudaFuncSetAttribute");
    set_to[{dev, fn}] = bytes;
    return 0;
}

Workspace workspace_layout(const tsa_desc& d) {
    Workspace w{};
    const size_t H = d.n_heads, L = d.seq_len, D = d.d_head;
    const size_t lq = lq_of(d);
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off = align_up(off + bytes, 256);
        return o;
    };
    w.status = take(4);
    w.k_keep = take(4);
    w.headsum = take(4 * L);
    w.logits = take(4 * H * lq * exact_logits_stride(d.seq_len));
    w.rowstat = take(score_fast_rowstat_bytes(d));
    w.rowmax = take(4 * H * lq);
    w.rowsum = take(4 * H * lq);
    w.colraw = take(4 * H * L);
    w.scores = take(4 * H * L);
    w.forced = take(4 * L);
    w.idx = take(4 * H * L);
    w.inv = take(4 * H * L);
    const size_t t = H * L * D * elem_bytes(d.dtype);
    w.qc = take(t);
    w.kc = take(t);
    w.vc = take(t);
    w.oc = take(t);
    w.total = off;
    return w;
}

namespace {

std::string fmt_double(double x) {
    char b[64];
    std::snprintf(b, sizeof b, "%f", x);
    return b;
}

int check_desc(const tsa_desc* d) {
    if (!d) return invalid("tsa: null descriptor");
    if (d->n_heads < 1 || d->n_kv_heads < 1 || d->n_heads % d->n_kv_heads != 0)
        return invalid("token_sparse_attention: " + std::to_string(d->n_heads) +
                       " query heads not divisible by " + std::to_string(d->n_kv_heads) +
                       " KV heads");
    if (d->seq_len < 1) return invalid("tsa: seq_len must be positive");
    if (d->dtype != TSA_F32 && d->dtype != TSA_BF16) return invalid("tsa: unknown dtype");
    const int D = d->d_head;
    if (D < 1 || D > 256)
        return invalid("tsa: unsupported d_head " + std::to_string(D) + " (supported: 1..256)");
    if (d->dtype == TSA_BF16 && D % 2 != 0)
        return invalid("tsa: bf16 rows need an even d_head, got " + std::to_string(D));
    if (d->last_q < 1)
        return invalid("score_tokens: last_q must be positive, got " + std::to_string(d->last_q));
    if (d->kernel < 1 || d->kernel % 2 == 0)
        return invalid("avg_pool_1d: kernel must be odd and positive, got " +
                       std::to_string(d->kernel));
    if (d->tau < 0.0 || d->tau > 1.0)
        return invalid("coverage_budget: tau " + fmt_double(d->tau) + " outside [0, 1]");
    if (d->s_fixed < 0.0 || d->s_fixed >= 1.0)
        return invalid("fixed_budget: sparsity ratio " + fmt_double(d->s_fixed) +
                       " outside [0, 1)");
    if (d->mode < TSA_MODE_DENSE || d->mode > TSA_MODE_FIXED) return invalid("tsa: unknown mode");
    if (d->forced_policy != TSA_FORCED_FINAL_TOKEN && d->forced_policy != TSA_FORCED_RECENT_WINDOW)
        return invalid("tsa: unknown forced policy");
    const int g = d->n_heads / d->n_kv_heads;
    if (d->head_begin < 0 || d->head_end > d->n_heads || d->head_begin >= d->head_end ||
        d->head_begin % g != 0 || d->head_end % g != 0)
        return invalid("tsa: head shard [" + std::to_string(d->head_begin) + ", " +
                       std::to_string(d->head_end) + ") is empty, out of range or splits a KV group");
    if (d->scoring == TSA_SCORING_FAST && d->dtype != TSA_BF16)
        return invalid("score_tokens: FAST scoring needs bf16 inputs");
    return 0;
}

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

template <typename T>
T* at(void* ws, size_t off) {
    return reinterpret_cast<T*>(static_cast<uint8_t*>(ws) + off);
}

// Forced set of SparsePlan::forced_set (model.cpp:74-79) as a suffix [fbegin, L).
int forced_begin(const tsa_desc& d) {
    if (d.forced_policy == TSA_FORCED_FINAL_TOKEN) return d.seq_len - 1;
    return std::max(0, d.seq_len - d.last_q);
}

int attend_dispatch(const tsa_desc& d, const void* q, const void* k, const void* v,
                    const int32_t* n_dev, int n_const, int kv_group, int rph, int kvrph, void* o,
                    cudaStream_t st) {
    if (attend_sm100_supported(d))
        return launch_attend_sm100(d, q, k, v, n_dev, n_const, kv_group, rph, kvrph, o, st);
    if (attend_tf32_supported(d))
        return launch_attend_tf32(d, q, k, v, n_dev, n_const, kv_group, rph, kvrph, o, st);
    return launch_attend_simt(d, q, k, v, n_dev, n_const, kv_group, rph, kvrph, o, st);
}

// f32 on the tensor cores: compress -> attend -> decompress with the decompress
// fused -- the gather also zeroes the output rows the selection dropped
// (scatter_rows' zero rows, tensor_ops.cpp:107) and the attention epilogue
// writes each kept row at its original position (idx), so there is no oc
// buffer and no scatter pass.  inv must be current (select / inverse).
static int sparse_attend_tf32(const tsa_desc& d, const void* q, const void* k, const void* v,
                              const int32_t* idx, const int32_t* k_keep, const int32_t* inv,
                              void* out, const Workspace& w, void* ws, cudaStream_t st) {
    int rc;
    if ((rc = launch_gather_zero(d, q, k, v, idx, k_keep, at<void>(ws, w.qc), at<void>(ws, w.kc),
                                 at<void>(ws, w.vc), inv, out, st)))
        return rc;
    return launch_attend_tf32(d, at<void>(ws, w.qc), at<void>(ws, w.kc), at<void>(ws, w.vc), k_keep,
                              d.seq_len, 1, d.seq_len, d.seq_len, out, st, idx);
}

int budget_impl(const tsa_desc& d, const float* s, int32_t* k_keep, void* ws, int min_keep,
                cudaStream_t st) {
    const Workspace w = workspace_layout(d);
    const int L = d.seq_len;
    if (min_keep < 1 || min_keep > L)
        return invalid("coverage_budget: min_keep " + std::to_string(min_keep) + " outside [1, " +
                       std::to_string(L) + "]");
    if (d.mode == TSA_MODE_DENSE) return launch_write_int(k_keep, L, st);
    if (d.mode == TSA_MODE_FIXED) {  // fixed_budget, token_coverage.cpp:98-109
        const int k = (int)std::lround((1.0 - d.s_fixed) * L);
        return launch_write_int(k_keep, std::max(k, min_keep), st);
    }
    return launch_budget(d, s, k_keep, at<float>(ws, w.headsum), at<int32_t>(ws, w.status),
                         min_keep, st);
}

}  // namespace

int forced_begin_of(const tsa_desc& d) { return forced_begin(d); }
int check_descriptor(const tsa_desc* d) { return check_desc(d); }
int budget_stage(const tsa_desc& d, const float* s, int32_t* k_keep, void* ws, int min_keep,
                 cudaStream_t st) {
    return budget_impl(d, s, k_keep, ws, min_keep, st);
}

int score_stage(const tsa_desc& d, const void* q, const void* k, const OutReplicas& s, void* ws,
                cudaStream_t st) {
    const Workspace w = workspace_layout(d);
    if (scoring_mode(d) == TSA_SCORING_FAST)
        return launch_score_fast(d, q, k, s, at<float>(ws, w.colraw), at<float>(ws, w.rowstat), st);
    if (score_exact_supported(d) && lq_of(d) <= 2048)
        return launch_score_exact(d, q, k, s, at<float>(ws, w.logits), at<int>(ws, w.rowmax),
                                  at<float>(ws, w.rowsum), at<float>(ws, w.colraw), st);
    return launch_score_reference(d, q, k, s, at<float>(ws, w.logits), at<int>(ws, w.rowmax),
                                  at<float>(ws, w.rowsum), at<float>(ws, w.colraw), st);
}

}  // namespace tsa

using namespace tsa;

extern "C" {

void tsa_desc_init(tsa_desc* d, int32_t n_heads, int32_t n_kv_heads, int32_t seq_len,
                   int32_t d_head, int32_t dtype) {
    d->n_heads = n_heads;
    d->n_kv_heads = n_kv_heads;
    d->seq_len = seq_len;
    d->d_head = d_head;
    d->dtype = dtype;
    d->mode = TSA_MODE_DYNAMIC;
    d->tau = 0.005;  // SparsePlan defaults, model.hpp:61-65
    d->s_fixed = 0.0;
    d->last_q = 64;
    d->kernel = 7;
    d->forced_policy = TSA_FORCED_FINAL_TOKEN;
    d->head_begin = 0;
    d->head_end = n_heads;
    d->scoring = TSA_SCORING_DEFAULT;
}

const char* tsa_last_error(void) { return tsa::g_error.c_str(); }

uint64_t tsa_kernel_launches(void) { return tsa::g_launches.load(); }

void tsa_release_graphs(void) { tsa::graph_cache_clear(); }

const char* tsa_version(void) { return "tsa_b200 0.1 (sm_100a)"; }

int tsa_workspace_size(const tsa_desc* d, size_t* bytes) {
    if (int rc = check_desc(d)) return rc;
    *bytes = workspace_layout(*d).total;
    return 0;
}

static int score_impl(const tsa_desc* d, const void* q, const void* k, const OutReplicas& s,
                      void* ws, void* stream) {
    return tsa::score_stage(*d, q, k, s, ws, S(stream));
}

int tsa_score(const tsa_desc* d, const void* q, const void* k, float* s, void* ws, void* stream) {
    if (int rc = check_desc(d)) return rc;
    return score_impl(d, q, k, single_replica(s), ws, stream);
}

static int make_replicas(const char* who, void* const* outs, int32_t n_outs, OutReplicas* r);

int tsa_expf(const float* x, float* y, int64_t n, void* stream) {
    if (n < 0 || (n > 0 && (!x || !y))) return invalid("tsa_expf: bad arguments");
    return launch_expf(x, y, n, S(stream));
}

int tsa_score_replicas(const tsa_desc* d, const void* q, const void* k, float* const* s_outs,
                       int32_t n_outs, void* ws, void* stream) {
    if (int rc = check_desc(d)) return rc;
    OutReplicas r;
    if (int rc = make_replicas("tsa_score_replicas", reinterpret_cast<void* const*>(s_outs),
                               n_outs, &r))
        return rc;
    return score_impl(d, q, k, r, ws, stream);
}

int tsa_budget(const tsa_desc* d, const float* s, int32_t* k_keep, void* ws, void* stream) {
    if (int rc = check_desc(d)) return rc;
    const int fb = forced_begin(*d);
    return budget_impl(*d, s, k_keep, ws, std::max(1, d->seq_len - fb), S(stream));
}

int tsa_aggregate_scores(const tsa_desc* d, const float* s, float* sl, void* ws, void* stream) {
    if (int rc = check_desc(d)) return rc;
    const Workspace w = workspace_layout(*d);
    return launch_aggregate(*d, s, sl, at<float>(ws, w.headsum), at<int32_t>(ws, w.status),
                            S(stream));
}

int tsa_coverage_budget(const tsa_desc* d, const float* sl, int32_t min_keep, int32_t* k_keep,
                        void* ws, void* stream) {
    if (int rc = check_desc(d)) return rc;
    if (min_keep < 1 || min_keep > d->seq_len)
        return invalid("coverage_budget: min_keep " + std::to_string(min_keep) + " outside [1, " +
                       std::to_string(d->seq_len) + "]");
    const Workspace w = workspace_layout(*d);
    return launch_coverage_from_sl(*d, sl, k_keep, at<int32_t>(ws, w.status), min_keep, S(stream));
}

int tsa_select(const tsa_desc* d, const float* s, const int32_t* k_keep, const int32_t* forced,
               int32_t n_forced, int32_t* idx, int32_t* inv, void* ws, void* stream) {
    if (int rc = check_desc(d)) return rc;
    (void)ws;
    if (n_forced < 0 || n_forced > d->seq_len) return invalid("select_tokens: bad forced count");
    if (n_forced > 0 && !forced) return invalid("select_tokens: null forced list");
    return launch_select(*d, s, k_keep, forced, n_forced, -1, idx, inv, S(stream));
}

int tsa_gather(const tsa_desc* d, const void* q, const void* k, const void* v, const int32_t* idx,
               const int32_t* k_keep, void* qc, void* kc, void* vc, void* stream) {
    if (int rc = check_desc(d)) return rc;
    if (!kc || !vc) return invalid("gather_rows: kc and vc are required (qc may be NULL)");
    return launch_gather(*d, q, k, v, idx, k_keep, qc, kc, vc, S(stream));
}

int tsa_attend(const tsa_desc* d, const void* qc, const void* kc, const void* vc,
               const int32_t* k_keep, int32_t kv_group, void* oc, void* stream) {
    if (int rc = check_desc(d)) return rc;
    if (kv_group < 1 || d->n_heads % kv_group != 0) return invalid("attend: bad kv_group");
    return attend_dispatch(*d, qc, kc, vc, k_keep, d->seq_len, kv_group, d->seq_len, d->seq_len,
                           oc, S(stream));
}

int tsa_scatter(const tsa_desc* d, const void* oc, const int32_t* inv, void* out, void* stream) {
    if (int rc = check_desc(d)) return rc;
    return launch_scatter(*d, oc, inv, out, S(stream));
}

int tsa_scatter_rows(const tsa_desc* d, const void* oc, const int32_t* idx, const int32_t* k_keep,
                     void* out, void* ws, void* stream) {
    if (int rc = check_desc(d)) return rc;
    const Workspace w = workspace_layout(*d);
    if (int rc = launch_inverse(*d, idx, k_keep, at<int32_t>(ws, w.inv), S(stream))) return rc;
    return launch_scatter(*d, oc, at<int32_t>(ws, w.inv), out, S(stream));
}

int tsa_attend_indexed(const tsa_desc* d, const void* q, const void* k, const void* v,
                       const void* kc, const void* vc, const int32_t* idx, const int32_t* k_keep,
                       void* out, void* stream) {
    if (int rc = check_desc(d)) return rc;
    if (!attend_sm100_supported(*d))
        return invalid("tsa_attend_indexed: the fused path needs bf16 and d_head 128");
    if (!q || !k || !v || !kc || !vc || !idx || !k_keep || !out)
        return invalid("tsa_attend_indexed: null buffer");
    return launch_attend_indexed(*d, q, k, v, kc, vc, idx, k_keep, out, S(stream));
}

int tsa_gather_zero(const tsa_desc* d, const void* k, const void* v, const int32_t* idx,
                    const int32_t* k_keep, void* kc, void* vc, const int32_t* inv, void* out,
                    void* stream) {
    if (int rc = check_desc(d)) return rc;
    if (!kc || !vc || !inv || !out) return invalid("tsa_gather_zero: null buffer");
    return launch_gather_zero(*d, nullptr, k, v, idx, k_keep, nullptr, kc, vc, inv, out, S(stream));
}

static int make_replicas(const char* who, void* const* outs, int32_t n_outs, OutReplicas* r) {
    if (!outs || n_outs < 1 || n_outs > TSA_MAX_REPLICAS)
        return invalid(std::string(who) + ": n_outs must be in [1, " +
                       std::to_string(TSA_MAX_REPLICAS) + "], got " + std::to_string(n_outs));
    *r = OutReplicas{};
    for (int i = 0; i < n_outs; ++i) {
        if (!outs[i]) return invalid(std::string(who) + ": null output replica " + std::to_string(i));
        r->p[i] = outs[i];
    }
    r->n = n_outs;
    return 0;
}

int tsa_gather_zero_replicas(const tsa_desc* d, const void* k, const void* v, const int32_t* idx,
                             const int32_t* k_keep, void* kc, void* vc, const int32_t* inv,
                             void* const* outs, int32_t n_outs, void* stream) {
    if (int rc = check_desc(d)) return rc;
    if (!kc || !vc || !inv) return invalid("tsa_gather_zero_replicas: null buffer");
    OutReplicas r;
    if (int rc = make_replicas("tsa_gather_zero_replicas", outs, n_outs, &r)) return rc;
    return launch_gather_zero_rep(*d, k, v, idx, k_keep, kc, vc, inv, r, S(stream));
}

int tsa_attend_indexed_replicas(const tsa_desc* d, const void* q, const void* k, const void* v,
                                const void* kc, const void* vc, const int32_t* idx,
                                const int32_t* k_keep, void* const* outs, int32_t n_outs,
                                void* stream) {
    if (int rc = check_desc(d)) return rc;
    if (!attend_sm100_supported(*d))
        return invalid("tsa_attend_indexed_replicas: the fused path needs bf16 and d_head 128");
    if (!q || !k || !v || !kc || !vc || !idx || !k_keep)
        return invalid("tsa_attend_indexed_replicas: null buffer");
    OutReplicas r;
    if (int rc = make_replicas("tsa_attend_indexed_replicas", outs, n_outs, &r)) return rc;
    return launch_attend_indexed_rep(*d, q, k, v, kc, vc, idx, k_keep, r, S(stream));
}

int tsa_zero_unselected(const tsa_desc* d, const int32_t* inv, void* out, void* stream) {
    if (int rc = check_desc(d)) return rc;
    return launch_zero_unselected(*d, inv, out, S(stream));
}

int tsa_check(const tsa_desc* d, void* ws, void* stream) {
    if (int rc = check_desc(d)) return rc;
    const Workspace w = workspace_layout(*d);
    int32_t status = 0;
    cudaError_t e = cudaMemcpyAsync(&status, at<int32_t>(ws, w.status), 4, cudaMemcpyDeviceToHost,
                                    S(stream));
    if (e == cudaSuccess) e = cudaStreamSynchronize(S(stream));
    if (e != cudaSuccess) return cuda_check(e, "tsa_check");
    if (status != 0) {
        cudaMemsetAsync(at<int32_t>(ws, w.status), 0, 4, S(stream));
        return invalid("aggregate_scores: all scores are zero, cannot normalize");
    }
    return 0;
}

int tsa_token_sparse_attention(const tsa_desc* d, const void* q, const void* k, const void* v,
                               const int32_t* idx, const int32_t* k_keep, void* out, void* ws,
                               void* stream) {
    if (int rc = check_desc(d)) return rc;
    const Workspace w = workspace_layout(*d);
    cudaStream_t st = S(stream);
    int rc;
    if (attend_sm100_supported(*d)) {  // fused gather -> attend -> scatter
        if ((rc = launch_inverse(*d, idx, k_keep, at<int32_t>(ws, w.inv), st))) return rc;
        if ((rc = launch_gather_zero(*d, q, k, v, idx, k_keep, nullptr, at<void>(ws, w.kc),
                                     at<void>(ws, w.vc), at<int32_t>(ws, w.inv), out, st)))
            return rc;
        return launch_attend_indexed(*d, q, k, v, at<void>(ws, w.kc), at<void>(ws, w.vc), idx,
                                     k_keep, out, st);
    }
    if (attend_tf32_supported(*d)) {
        if ((rc = launch_inverse(*d, idx, k_keep, at<int32_t>(ws, w.inv), st))) return rc;
        return sparse_attend_tf32(*d, q, k, v, idx, k_keep, at<int32_t>(ws, w.inv), out, w, ws, st);
    }
    if ((rc = launch_gather(*d, q, k, v, idx, k_keep, at<void>(ws, w.qc), at<void>(ws, w.kc),
                            at<void>(ws, w.vc), st)))
        return rc;
    if ((rc = attend_dispatch(*d, at<void>(ws, w.qc), at<void>(ws, w.kc), at<void>(ws, w.vc), k_keep,
                              d->seq_len, 1, d->seq_len, d->seq_len, at<void>(ws, w.oc), st)))
        return rc;
    if ((rc = launch_inverse(*d, idx, k_keep, at<int32_t>(ws, w.inv), st))) return rc;
    return launch_scatter(*d, at<void>(ws, w.oc), at<int32_t>(ws, w.inv), out, st);
}

int tsa_dense_attention(const tsa_desc* d, const void* q, const void* k, const void* v, void* out,
                        void* stream) {
    if (int rc = check_desc(d)) return rc;
    return attend_dispatch(*d, q, k, v, nullptr, d->seq_len, d->n_heads / d->n_kv_heads,
                           d->seq_len, d->seq_len, out, S(stream));
}

static int layer_eager(const tsa_desc* d, const void* q, const void* k, const void* v,
                               void* out, int32_t* idx_out, int32_t* k_keep_out,
                               int32_t* k_keep_host, void* ws, cudaStream_t st) {
    void* stream = st;
    int rc;
    if (d->mode == TSA_MODE_DENSE) {
        if ((rc = launch_write_int(k_keep_out, d->seq_len, st))) return rc;
        if ((rc = tsa_dense_attention(d, q, k, v, out, stream))) return rc;
    } else {
        const Workspace w = workspace_layout(*d);
        float* s = at<float>(ws, w.scores);
        int32_t* idx = idx_out ? idx_out : at<int32_t>(ws, w.idx);
        int32_t* inv = at<int32_t>(ws, w.inv);
        const int fb = forced_begin(*d);
        const int nf = d->seq_len - fb;
        if ((rc = tsa_score(d, q, k, s, ws, stream))) return rc;
        if ((rc = budget_impl(*d, s, k_keep_out, ws, std::max(1, nf), st))) return rc;
        if ((rc = launch_select(*d, s, k_keep_out, nullptr, nf, fb, idx, inv, st))) return rc;
        if (attend_sm100_supported(*d)) {  // K/V gather + zero-fill, then fused Q-gather/attend/scatter
            if ((rc = launch_gather_zero(*d, q, k, v, idx, k_keep_out, nullptr, at<void>(ws, w.kc),
                                         at<void>(ws, w.vc), inv, out, st)))
                return rc;
            if ((rc = launch_attend_indexed(*d, q, k, v, at<void>(ws, w.kc), at<void>(ws, w.vc), idx,
                                            k_keep_out, out, st)))
                return rc;
        } else if (attend_tf32_supported(*d)) {
            if ((rc = sparse_attend_tf32(*d, q, k, v, idx, k_keep_out, inv, out, w, ws, st))) return rc;
        } else {
        if ((rc = launch_gather(*d, q, k, v, idx, k_keep_out, at<void>(ws, w.qc), at<void>(ws, w.kc),
                                at<void>(ws, w.vc), st)))
            return rc;
        if ((rc = attend_dispatch(*d, at<void>(ws, w.qc), at<void>(ws, w.kc), at<void>(ws, w.vc),
                                  k_keep_out, d->seq_len, 1, d->seq_len, d->seq_len,
                                  at<void>(ws, w.oc), st)))
            return rc;
        if ((rc = launch_scatter(*d, at<void>(ws, w.oc), inv, out, st))) return rc;
        }
    }
    if (k_keep_host) {
        cudaError_t e = cudaMemcpyAsync(k_keep_host, k_keep_out, 4, cudaMemcpyDeviceToHost, st);
        if (e != cudaSuccess) return cuda_check(e, "k_keep copy");
    }
    return 0;
}

int tsa_sparse_attention_layer(const tsa_desc* d, const void* q, const void* k, const void* v,
                               void* out, int32_t* idx_out, int32_t* k_keep_out,
                               int32_t* k_keep_host, void* ws, void* stream) {
    if (int rc = check_desc(d)) return rc;
    if (!k_keep_out) return invalid("tsa_sparse_attention_layer: k_keep_out is required");
    return tsa::graph_launch(*d, {q, k, v, out, idx_out, k_keep_out, k_keep_host, ws}, S(stream),
                             [&](cudaStream_t st) {
                                 return layer_eager(d, q, k, v, out, idx_out, k_keep_out,
                                                    k_keep_host, ws, st);
                             });
}

// ---- host-buffer entry point: the layer with its transfers pipelined ----
// q/k/v/out_host are the caller's host tensors (pinned for asynchronous copies);
// q/k/v/out are device staging buffers of the same shapes.  K and the Q tail
// rows go first (scoring needs all of them), then each head group's V heads
// and remaining Q rows on a copy stream while the compute stream scores and
// selects; compress + attention then run per head group, each waiting only for
// its own rows, and every finished group's output rows are copied back on a
// second copy stream while the next group computes.
namespace {
struct HostPipe {
    cudaStream_t in = nullptr, out = nullptr;
    cudaEvent_t start = nullptr, kvq = nullptr, q[64] = {}, done[64] = {}, vr[64] = {},
                kr[64] = {}, fin = nullptr;
};
// One pipeline (copy streams + events) per calling thread and device: two
// threads' host-tensor calls never share streams or events (the reference's
// operators are pure and safe to call concurrently).
HostPipe* host_pipe(int device) {
    thread_local HostPipe pipes[16];
    thread_local bool init[16] = {};
    if (device < 0 || device >= 16) return nullptr;
    HostPipe& p = pipes[device];
    if (!init[device]) {
        const unsigned f = cudaEventDisableTiming;
        if (cudaStreamCreateWithFlags(&p.in, cudaStreamNonBlocking) != cudaSuccess ||
            cudaStreamCreateWithFlags(&p.out, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&p.start, f) != cudaSuccess ||
            cudaEventCreateWithFlags(&p.kvq, f) != cudaSuccess ||
            cudaEventCreateWithFlags(&p.fin, f) != cudaSuccess)
            return nullptr;
        for (int g = 0; g < 64; ++g)
            if (cudaEventCreateWithFlags(&p.q[g], f) != cudaSuccess ||
                cudaEventCreateWithFlags(&p.done[g], f) != cudaSuccess ||
                cudaEventCreateWithFlags(&p.vr[g], f) != cudaSuccess ||
                cudaEventCreateWithFlags(&p.kr[g], f) != cudaSuccess)
                return nullptr;
        init[device] = true;
    }
    return &p;
}
}  // namespace

int tsa_sparse_attention_layer_host(const tsa_desc* d, const void* q_host, const void* k_host,
                                    const void* v_host, void* out_host, void* q, void* k, void* v,
                                    void* out, int32_t* idx_out, int32_t* k_keep_out,
                                    int32_t* k_keep_host, void* ws, int32_t n_groups,
                                    void* stream) {
    if (int rc = check_desc(d)) return rc;
    if (!q_host || !k_host || !v_host || !out_host || !q || !k || !v || !out || !k_keep_out)
        return invalid("tsa_sparse_attention_layer_host: null pointer");
    if (d->head_begin != 0 || d->head_end != d->n_heads)
        return invalid("tsa_sparse_attention_layer_host: the whole layer (no head shard)");
    cudaStream_t st = S(stream);
    const size_t eb = elem_bytes(d->dtype), L = d->seq_len, D = d->d_head;
    const size_t head_bytes = L * D * eb;
    const int H = d->n_heads, Hkv = d->n_kv_heads, g = H / Hkv;
    cudaError_t e;
#define TSA_HCK(x)                                                          \
    do {                                                                    \
        if ((e = (x)) != cudaSuccess) return cuda_check(e, "layer_host");   \
    } while (0)
    const bool pipelined = attend_sm100_supported(*d) && d->mode != TSA_MODE_DENSE;
    if (!pipelined) {  // one copy in, the layer, one copy out
        TSA_HCK(cudaMemcpyAsync(q, q_host, H * head_bytes, cudaMemcpyHostToDevice, st));
        TSA_HCK(cudaMemcpyAsync(k, k_host, Hkv * head_bytes, cudaMemcpyHostToDevice, st));
        TSA_HCK(cudaMemcpyAsync(v, v_host, Hkv * head_bytes, cudaMemcpyHostToDevice, st));
        if (int rc = tsa_sparse_attention_layer(d, q, k, v, out, idx_out, k_keep_out, k_keep_host,
                                                ws, stream))
            return rc;
        TSA_HCK(cudaMemcpyAsync(out_host, out, H * head_bytes, cudaMemcpyDeviceToHost, st));
        return 0;
    }
    int dev = 0;
    TSA_HCK(cudaGetDevice(&dev));
    HostPipe* p = host_pipe(dev);
    if (!p) return cuda_check(cudaGetLastError(), "layer_host: streams");
    // groups of whole KV groups
    int G = n_groups > 0 ? n_groups : Hkv;
    G = std::max(1, std::min({G, Hkv, 64}));
    while (Hkv % G) --G;
    const int hpg = H / G;  // query heads per group
    const size_t lq = lq_of(*d);
    auto* qd = static_cast<uint8_t*>(q);
    auto* qh = static_cast<const uint8_t*>(q_host);
    TSA_HCK(cudaEventRecord(p->start, st));  // the device buffers are free after prior work
    TSA_HCK(cudaStreamWaitEvent(p->in, p->start, 0));
    TSA_HCK(cudaStreamWaitEvent(p->out, p->start, 0));
    // scoring inputs first: the Q tail rows of every head, then K two KV heads at
    // a time -- their scoring starts as soon as their K rows have arrived, so all
    // but the last pair's scoring hides under the K copy
    const size_t tail_off = (L - lq) * D * eb;
    TSA_HCK(cudaMemcpy2DAsync(qd + tail_off, head_bytes, qh + tail_off, head_bytes, lq * D * eb, H,
                              cudaMemcpyHostToDevice, p->in));
    // two KV heads per scoring launch: each launch's row-sum chain costs its full
    // L-long latency, so one launch per KV head would fall behind the copy
    const int score_groups = Hkv > 64 ? 1 : (Hkv % 2 == 0 ? Hkv / 2 : Hkv);
    for (int i = 0; i < score_groups; ++i) {
        const size_t kv0 = (size_t)i * (Hkv / score_groups), nkv = Hkv / score_groups;
        TSA_HCK(cudaMemcpyAsync(static_cast<uint8_t*>(k) + kv0 * head_bytes,
                                static_cast<const uint8_t*>(k_host) + kv0 * head_bytes,
                                nkv * head_bytes, cudaMemcpyHostToDevice, p->in));
        TSA_HCK(cudaEventRecord(p->kr[i], p->in));
    }
    // Compute chunks: one query head each (a group's K/V are compressed once, before
    // its first head) -- an attention waits for one head's Q rows, not a group's,
    // so the copies stay ahead of the compute after the first group (whole groups
    // left the compute idle at every group boundary), and the last copy back is
    // one head's rows.  More than 64 heads: whole groups, the ends head by head.
    struct Chunk { int h0, h1, gi; };
    Chunk chunks[64];
    int nc = 0;
    const bool per_head = H <= 64;
    const bool split_ends = G >= 2 && hpg > 1 && (G - 2) + 2 * hpg <= 64;
    for (int gi = 0; gi < G; ++gi) {
        if (per_head || (split_ends && (gi == 0 || gi == G - 1)))
            for (int h = gi * hpg; h < (gi + 1) * hpg; ++h) chunks[nc++] = {h, h + 1, gi};
        else
            chunks[nc++] = {gi * hpg, (gi + 1) * hpg, gi};
    }
    // then, group by group, the group's V heads and the rest of its Q rows (per chunk)
    const int kvpg = Hkv / G;
    for (int c = 0, gi_done = -1; c < nc; ++c) {
        const int gi = chunks[c].gi;
        if (gi != gi_done) {
            const size_t kv0 = (size_t)gi * kvpg;
            TSA_HCK(cudaMemcpyAsync(static_cast<uint8_t*>(v) + kv0 * head_bytes,
                                    static_cast<const uint8_t*>(v_host) + kv0 * head_bytes,
                                    (size_t)kvpg * head_bytes, cudaMemcpyHostToDevice, p->in));
            TSA_HCK(cudaEventRecord(p->vr[gi], p->in));
            gi_done = gi;
        }
        const size_t h0 = chunks[c].h0, nh = chunks[c].h1 - chunks[c].h0;
        if (L > lq)
            TSA_HCK(cudaMemcpy2DAsync(qd + h0 * head_bytes, head_bytes, qh + h0 * head_bytes,
                                      head_bytes, (L - lq) * D * eb, nh, cudaMemcpyHostToDevice,
                                      p->in));
        TSA_HCK(cudaEventRecord(p->q[c], p->in));
    }
    // score (KV group by KV group, as K arrives) -> budget -> select on the compute stream
    const Workspace w = workspace_layout(*d);
    float* s = at<float>(ws, w.scores);
    int32_t* idx = idx_out ? idx_out : at<int32_t>(ws, w.idx);
    int32_t* inv = at<int32_t>(ws, w.inv);
    const int fb = forced_begin(*d);
    const int nf = d->seq_len - fb;
    int rc;
    for (int i = 0; i < score_groups; ++i) {
        tsa_desc ds = *d;
        ds.head_begin = i * (H / score_groups);
        ds.head_end = (i + 1) * (H / score_groups);
        TSA_HCK(cudaStreamWaitEvent(st, p->kr[i], 0));
        if ((rc = tsa_score(&ds, q, k, s, ws, stream))) return rc;
    }
    if ((rc = budget_impl(*d, s, k_keep_out, ws, std::max(1, nf), st))) return rc;
    if ((rc = launch_select(*d, s, k_keep_out, nullptr, nf, fb, idx, inv, st))) return rc;
    // per chunk: compress K/V of its group (+ zero the group's dropped rows) once,
    // attend, and stream the chunk's output rows back while the next one computes
    for (int c = 0, gi_done = -1; c < nc; ++c) {
        const int gi = chunks[c].gi;
        if (gi != gi_done) {
            tsa_desc dg = *d;
            dg.head_begin = gi * hpg;
            dg.head_end = (gi + 1) * hpg;
            TSA_HCK(cudaStreamWaitEvent(st, p->vr[gi], 0));
            if ((rc = launch_gather_zero(dg, q, k, v, idx, k_keep_out, nullptr, at<void>(ws, w.kc),
                                         at<void>(ws, w.vc), inv, out, st)))
                return rc;
            gi_done = gi;
        }
        tsa_desc dc = *d;
        dc.head_begin = chunks[c].h0;
        dc.head_end = chunks[c].h1;
        TSA_HCK(cudaStreamWaitEvent(st, p->q[c], 0));
        if ((rc = launch_attend_indexed(dc, q, k, v, at<void>(ws, w.kc), at<void>(ws, w.vc), idx,
                                        k_keep_out, out, st)))
            return rc;
        TSA_HCK(cudaEventRecord(p->done[c], st));
        TSA_HCK(cudaStreamWaitEvent(p->out, p->done[c], 0));
        TSA_HCK(cudaMemcpyAsync(static_cast<uint8_t*>(out_host) + (size_t)dc.head_begin * head_bytes,
                                static_cast<uint8_t*>(out) + (size_t)dc.head_begin * head_bytes,
                                (size_t)(dc.head_end - dc.head_begin) * head_bytes,
                                cudaMemcpyDeviceToHost, p->out));
    }
    if (k_keep_host)
        TSA_HCK(cudaMemcpyAsync(k_keep_host, k_keep_out, 4, cudaMemcpyDeviceToHost, st));
    TSA_HCK(cudaEventRecord(p->fin, p->out));
    TSA_HCK(cudaStreamWaitEvent(st, p->fin, 0));  // completion on `stream` covers the copies
#undef TSA_HCK
    (void)g;
    return 0;
}

// ---- attention-branch producer / consumer (cfg4 stack) ----
int tsa_rms_norm(const void* x, const float* gain, int64_t rows, int32_t cols, float eps,
                 int32_t dtype, void* out, void* stream) {
    if (rows < 0 || cols < 1) return invalid("rms_norm: bad shape");
    if (dtype != TSA_F32 && dtype != TSA_BF16) return invalid("rms_norm: unknown dtype");
    if (!x || !gain || !out) return invalid("rms_norm: null pointer");
    if (rows == 0) return 0;
    return launch_rms_norm(x, gain, rows, cols, eps, dtype, out, S(stream));
}

int tsa_rope_table(int32_t seq_len, int32_t d_head, float theta, float* table, void* stream) {
    if (d_head % 2 != 0)
        return invalid("apply_rope: odd head dimension " + std::to_string(d_head));
    if (seq_len < 1 || !table) return invalid("rope_table: bad arguments");
    return launch_rope_table(seq_len, d_head, theta, table, S(stream));
}

int tsa_split_heads_rope(const tsa_desc* d, const void* qkv, const float* table, void* q, void* k,
                         void* v, void* stream) {
    if (int rc = check_desc(d)) return rc;
    if (d->d_head % 2 != 0)
        return invalid("apply_rope: odd head dimension " + std::to_string(d->d_head));
    if (!qkv || !table || !q || !k || !v) return invalid("split_heads_rope: null pointer");
    return launch_split_heads_rope(*d, qkv, table, q, k, v, S(stream));
}

int tsa_heads_concat(const tsa_desc* d, const void* heads, void* cat, void* stream) {
    if (int rc = check_desc(d)) return rc;
    if (!heads || !cat) return invalid("heads_concat: null pointer");
    return launch_heads_concat(*d, heads, cat, S(stream));
}

// ---- the projections on the tensor cores (proj_gemm.cu) ----
int tsa_gemm_bf16(const void* a, const void* b_t, void* c, int32_t M, int32_t N, int32_t K,
                  void* stream) {
    if (!a || !b_t || !c) return invalid("gemm_bf16: null pointer");
    return launch_gemm_bf16(a, b_t, c, M, N, K, S(stream));
}

int tsa_prepare_weight(const void* w, int32_t dtype, const float* gain, int32_t rows, int32_t cols,
                       void* w_t, void* stream) {
    if (!w || !w_t) return invalid("prepare_weight: null pointer");
    if (rows < 1 || cols < 1) return invalid("prepare_weight: bad shape");
    if (dtype != TSA_F32 && dtype != TSA_BF16) return invalid("prepare_weight: unknown dtype");
    return launch_prepare_weight(w, dtype, gain, rows, cols, w_t, S(stream));
}

int tsa_row_inv_rms(const void* x, int64_t rows, int32_t cols, float eps, float* inv, void* stream) {
    if (!x || !inv) return invalid("row_inv_rms: null pointer");
    if (rows < 0 || cols < 1) return invalid("row_inv_rms: bad shape");
    return launch_row_inv_rms(x, rows, cols, eps, inv, S(stream));
}

int tsa_qkv_proj(const tsa_desc* d, const void* x, int32_t d_model, const void* w_t,
                 const float* inv_rms, const float* table, void* q, void* k, void* v, void* stream) {
    if (int rc = check_desc(d)) return rc;
    if (!x || !w_t || !table || !q || !k || !v) return invalid("qkv_proj: null pointer");
    return launch_qkv_proj(*d, x, d_model, w_t, inv_rms, table, q, k, v, S(stream));
}

int tsa_out_proj_residual(const tsa_desc* d, const void* o, const void* wo_t, int32_t d_model,
                          void* x, void* stream) {
    if (int rc = check_desc(d)) return rc;
    if (!o || !wo_t || !x) return invalid("out_proj_residual: null pointer");
    return launch_out_proj_residual(*d, o, wo_t, d_model, x, S(stream));
}

// ---- drift calibration (drift.cpp:14-65) ----
int tsa_layer_drift(const void* prev, const void* next, int64_t rows, int32_t cols, int32_t dtype,
                    double epsilon, double* r_out, void* ws, void* stream) {
    if (!(epsilon > 0)) return invalid("compute_drift: epsilon must be positive");
    if (rows < 1 || cols < 1 || !prev || !next || !r_out || !ws)
        return invalid("compute_drift: bad arguments");
    if (dtype != TSA_F32 && dtype != TSA_BF16) return invalid("compute_drift: unknown dtype");
    return launch_layer_drift(prev, next, rows, cols, dtype, epsilon, r_out,
                              static_cast<double*>(ws), S(stream));
}

int tsa_select_sparse_layers(const double* R, int32_t n, double delta, double* R_hat,
                             int32_t* layers, int32_t* n_layers) {
    if (n < 1 || !R) return invalid("select_sparse_layers: empty drift vector");
    int m = 0;
    for (int l = 0; l < n; ++l) {
        int count = 0;
        for (int k = 0; k < n; ++k)
            if (R[k] <= R[l]) ++count;
        const double rh = static_cast<double>(count) / static_cast<double>(n);
        if (R_hat) R_hat[l] = rh;
        if (rh <= delta && layers) layers[m] = l;
        if (rh <= delta) ++m;
    }
    if (n_layers) *n_layers = m;
    return 0;
}

}  // extern "C"
