// Defines the reference's operator functions (namespace tsa) on the B200 C
// ABI.  See include/tsa_b200.hpp for the mapping and INTEGRATION.md for the
// build change.  Host <-> device traffic is per call (the reference API is
// host-memory based); production callers use the C ABI with device buffers.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "tsa/attention.hpp"
#include "tsa/selection.hpp"
#include "tsa/token_coverage.hpp"
#include "tsa_b200.hpp"

namespace tsa {
namespace b200 {
namespace {

int g_device = 0;
int g_scoring = TSA_SCORING_REFERENCE;

void check(int rc) {
    if (rc == TSA_OK) return;
    const std::string msg = tsa_last_error();
    if (rc == TSA_ERR_INVALID) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

void cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// Device buffer owning RAII.
struct Dev {
    void* p = nullptr;
    size_t n = 0;
    explicit Dev(size_t bytes) : n(bytes) {
        cuda(cudaSetDevice(g_device), "cudaSetDevice");
        cuda(cudaMalloc(&p, std::max<size_t>(bytes, 16)), "cudaMalloc");
    }
    ~Dev() { cudaFree(p); }
    Dev(const Dev&) = delete;
    Dev& operator=(const Dev&) = delete;
    Dev(Dev&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; }
    template <typename T>
    T* as() const { return static_cast<T*>(p); }
    void upload(const void* src, size_t bytes, size_t off = 0) {
        cuda(cudaMemcpy(static_cast<char*>(p) + off, src, bytes, cudaMemcpyHostToDevice), "H2D");
    }
    void download(void* dst, size_t bytes, size_t off = 0) const {
        cuda(cudaMemcpy(dst, static_cast<const char*>(p) + off, bytes, cudaMemcpyDeviceToHost), "D2H");
    }
};

void upload_heads(Dev& d, const std::vector<Matrix>& ms, size_t per) {
    for (size_t h = 0; h < ms.size(); ++h)
        if (per) d.upload(ms[h].data(), per * sizeof(float), h * per * sizeof(float));
}

tsa_desc make_desc(int H, int Hkv, int L, int d) {
    tsa_desc desc;
    tsa_desc_init(&desc, H, Hkv, L, d, TSA_F32);
    desc.scoring = g_scoring;
    return desc;
}

Dev workspace(const tsa_desc& d) {
    size_t bytes = 0;
    check(tsa_workspace_size(&d, &bytes));
    Dev ws(bytes);
    cuda(cudaMemset(ws.p, 0, bytes), "memset");
    return ws;
}

// Scores-only descriptor (the budget/selection calls ignore d/dtype).
tsa_desc scores_desc(int H, int L) {
    tsa_desc d = make_desc(H, 1, L, 8);
    d.last_q = 1;
    return d;
}

void check_heads(const HeadTensors& heads) {
    const int H = heads.n_heads(), Hkv = heads.n_kv_heads();
    if (H == 0 || Hkv == 0 || H % Hkv != 0)
        throw std::invalid_argument("token_sparse_attention: " + std::to_string(H) +
                                    " query heads not divisible by " + std::to_string(Hkv) +
                                    " KV heads");
}

}  // namespace

void set_device(int device) { g_device = device; }
void set_scoring(int scoring) { g_scoring = scoring; }

}  // namespace b200

using namespace b200;

// token_coverage.hpp:32
HeadScores score_tokens(const HeadTensors& heads, int last_q, int kernel) {
    if (last_q < 1)
        throw std::invalid_argument("score_tokens: last_q must be positive, got " +
                                    std::to_string(last_q));
    check_heads(heads);
    const int H = heads.n_heads(), Hkv = heads.n_kv_heads();
    const int L = static_cast<int>(heads.q[0].rows()), d = static_cast<int>(heads.q[0].cols());
    tsa_desc desc = make_desc(H, Hkv, L, d);
    desc.last_q = last_q;
    desc.kernel = kernel;
    const size_t per = size_t(L) * size_t(d);
    Dev q(sizeof(float) * H * per), k(sizeof(float) * Hkv * per), s(sizeof(float) * H * L);
    upload_heads(q, heads.q, per);
    upload_heads(k, heads.k, per);
    Dev ws = workspace(desc);
    check(tsa_score(&desc, q.p, k.p, s.as<float>(), ws.p, nullptr));
    cuda(cudaDeviceSynchronize(), "score_tokens");
    HeadScores hs;
    hs.s.resize(H, L);
    s.download(hs.s.data(), sizeof(float) * H * L);
    hs.last_q = std::min(last_q, L);
    hs.kernel = kernel;
    return hs;
}

// token_coverage.hpp:36
LayerScores aggregate_scores(const HeadScores& hs) {
    const int H = static_cast<int>(hs.s.rows()), L = static_cast<int>(hs.s.cols());
    tsa_desc desc = scores_desc(H, L);
    Dev s(sizeof(float) * H * L), sl(sizeof(float) * L);
    s.upload(hs.s.data(), sizeof(float) * H * L);
    Dev ws = workspace(desc);
    check(tsa_aggregate_scores(&desc, s.as<float>(), sl.as<float>(), ws.p, nullptr));
    check(tsa_check(&desc, ws.p, nullptr));
    LayerScores out;
    out.s.resize(L);
    sl.download(out.s.data(), sizeof(float) * L);
    return out;
}

// token_coverage.hpp:42
int coverage_budget(const LayerScores& sl, double tau, int min_keep) {
    const int L = static_cast<int>(sl.s.size());
    tsa_desc desc = scores_desc(1, L);
    desc.tau = tau;
    Dev s(sizeof(float) * L), k(sizeof(int32_t));
    s.upload(sl.s.data(), sizeof(float) * L);
    Dev ws = workspace(desc);
    check(tsa_coverage_budget(&desc, s.as<float>(), min_keep, k.as<int32_t>(), ws.p, nullptr));
    int32_t kk = 0;
    k.download(&kk, sizeof(kk));
    return kk;
}

// token_coverage.hpp:45 (integer arithmetic, host side as in the reference)
int fixed_budget(int seq_len, double s, int min_keep) {
    if (s < 0.0 || s >= 1.0)
        throw std::invalid_argument("fixed_budget: sparsity ratio " + std::to_string(s) +
                                    " outside [0, 1)");
    if (min_keep < 1 || min_keep > seq_len)
        throw std::invalid_argument("fixed_budget: min_keep " + std::to_string(min_keep) +
                                    " outside [1, " + std::to_string(seq_len) + "]");
    const int k = static_cast<int>(std::lround((1.0 - s) * seq_len));
    return std::max(k, min_keep);
}

// token_coverage.hpp:50
TokenSelection select_tokens(const HeadScores& hs, int k_keep, const IndexList& forced) {
    const int H = static_cast<int>(hs.s.rows()), L = static_cast<int>(hs.s.cols());
    IndexList f = forced;  // normalised as the reference does (token_coverage.cpp:113-121)
    std::sort(f.begin(), f.end());
    f.erase(std::unique(f.begin(), f.end()), f.end());
    for (int t : f)
        if (t < 0 || t >= L)
            throw std::invalid_argument("select_tokens: forced index " + std::to_string(t) +
                                        " out of range [0, " + std::to_string(L) + ")");
    const int min_keep = std::max<int>(1, static_cast<int>(f.size()));
    if (k_keep < min_keep || k_keep > L)
        throw std::invalid_argument("select_tokens: k_keep " + std::to_string(k_keep) +
                                    " outside [" + std::to_string(min_keep) + ", " +
                                    std::to_string(L) + "]");
    tsa_desc desc = scores_desc(H, L);
    Dev s(sizeof(float) * H * L), idx(sizeof(int32_t) * H * L), kd(sizeof(int32_t)),
        fd(sizeof(int32_t) * std::max<size_t>(1, f.size()));
    s.upload(hs.s.data(), sizeof(float) * H * L);
    const int32_t kk = k_keep;
    kd.upload(&kk, sizeof(kk));
    if (!f.empty()) fd.upload(f.data(), sizeof(int32_t) * f.size());
    Dev ws = workspace(desc);
    check(tsa_select(&desc, s.as<float>(), kd.as<int32_t>(), fd.as<int32_t>(),
                     static_cast<int32_t>(f.size()), idx.as<int32_t>(), nullptr, ws.p, nullptr));
    std::vector<int32_t> host(size_t(H) * L);
    idx.download(host.data(), sizeof(int32_t) * host.size());
    TokenSelection sel;
    sel.k_keep = k_keep;
    sel.forced = f;
    sel.indices.resize(size_t(H));
    for (int h = 0; h < H; ++h)
        sel.indices[size_t(h)].assign(host.begin() + size_t(h) * L,
                                      host.begin() + size_t(h) * L + k_keep);
    return sel;
}

// attention.hpp:31
Matrix dense_causal_attention(const Matrix& q, const Matrix& k, const Matrix& v) {
    if (q.cols() != k.cols() || k.rows() != v.rows() || k.cols() != q.cols())
        throw std::invalid_argument("attention: inconsistent head shapes Q" + shape_str(q) + " K" +
                                    shape_str(k) + " V" + shape_str(v));
    if (q.rows() != k.rows())
        throw std::invalid_argument("dense_causal_attention: Q" + shape_str(q) + " and K" +
                                    shape_str(k) + " disagree on length");
    const int n = static_cast<int>(q.rows()), d = static_cast<int>(q.cols());
    Matrix out(n, v.cols());
    if (n == 0) return out;
    tsa_desc desc = make_desc(1, 1, n, d);
    const size_t bytes = sizeof(float) * size_t(n) * size_t(d);
    Dev dq(bytes), dk(bytes), dv(bytes), dout(bytes);
    dq.upload(q.data(), bytes);
    dk.upload(k.data(), bytes);
    dv.upload(v.data(), bytes);
    check(tsa_dense_attention(&desc, dq.p, dk.p, dv.p, dout.p, nullptr));
    cuda(cudaDeviceSynchronize(), "dense_causal_attention");
    dout.download(out.data(), bytes);
    return out;
}

// attention.hpp:44-45
std::vector<Matrix> token_sparse_attention(const HeadTensors& heads, const TokenSelection& sel,
                                           const AttentionKernel& inner) {
    check_heads(heads);
    const int H = heads.n_heads(), Hkv = heads.n_kv_heads();
    if (static_cast<int>(sel.indices.size()) != H)
        throw std::invalid_argument("token_sparse_attention: selection covers " +
                                    std::to_string(sel.indices.size()) + " heads, tensors have " +
                                    std::to_string(H));
    const int L = static_cast<int>(heads.q[0].rows()), d = static_cast<int>(heads.q[0].cols());
    validate(sel, L);  // the reference's own check (selection.cpp:12-45)
    const int k = sel.k_keep;
    tsa_desc desc = make_desc(H, Hkv, L, d);
    const size_t per = size_t(L) * size_t(d);
    Dev q(sizeof(float) * H * per), kt(sizeof(float) * Hkv * per), v(sizeof(float) * Hkv * per),
        out(sizeof(float) * H * per), idx(sizeof(int32_t) * H * L), kd(sizeof(int32_t));
    upload_heads(q, heads.q, per);
    upload_heads(kt, heads.k, per);
    upload_heads(v, heads.v, per);
    std::vector<int32_t> flat(size_t(H) * L, 0);
    for (int h = 0; h < H; ++h)
        std::copy(sel.indices[size_t(h)].begin(), sel.indices[size_t(h)].end(),
                  flat.begin() + size_t(h) * L);
    idx.upload(flat.data(), sizeof(int32_t) * flat.size());
    const int32_t kk = k;
    kd.upload(&kk, sizeof(kk));
    Dev ws = workspace(desc);
    // the default argument (attention.hpp:45) wraps this library's own
    // dense_causal_attention: run the whole operator on the GPU then
    using Fn = Matrix (*)(const Matrix&, const Matrix&, const Matrix&);
    const Fn* fp = inner ? inner.target<Fn>() : nullptr;
    const bool default_inner = !inner || (fp && *fp == &dense_causal_attention);
    if (default_inner) {
        check(tsa_token_sparse_attention(&desc, q.p, kt.p, v.p, idx.as<int32_t>(), kd.as<int32_t>(),
                                         out.p, ws.p, nullptr));
    } else {
        // the AttentionKernel seam (attention.hpp:28): gather on the GPU, call
        // the caller's kernel once per head on k x d tensors, scatter back
        Dev qc(sizeof(float) * H * per), kc(sizeof(float) * H * per), vc(sizeof(float) * H * per),
            oc(sizeof(float) * H * per);
        check(tsa_gather(&desc, q.p, kt.p, v.p, idx.as<int32_t>(), kd.as<int32_t>(), qc.p, kc.p,
                         vc.p, nullptr));
        cuda(cudaDeviceSynchronize(), "gather");
        for (int h = 0; h < H; ++h) {
            Matrix mq(k, d), mk(k, d), mv(k, d);
            const size_t off = sizeof(float) * size_t(h) * per, b = sizeof(float) * size_t(k) * d;
            qc.download(mq.data(), b, off);
            kc.download(mk.data(), b, off);
            vc.download(mv.data(), b, off);
            const Matrix r = inner(mq, mk, mv);
            if (r.rows() != k || r.cols() != d)
                throw std::invalid_argument("token_sparse_attention: inner returned " + shape_str(r));
            oc.upload(r.data(), b, off);
        }
        check(tsa_scatter_rows(&desc, oc.p, idx.as<int32_t>(), kd.as<int32_t>(), out.p, ws.p,
                               nullptr));
    }
    cuda(cudaDeviceSynchronize(), "token_sparse_attention");
    std::vector<Matrix> res(size_t(H), Matrix(L, d));
    for (int h = 0; h < H; ++h)
        out.download(res[size_t(h)].data(), sizeof(float) * per, sizeof(float) * size_t(h) * per);
    return res;
}

}  // namespace tsa
