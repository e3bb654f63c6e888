// ref_capi.cpp -- C entry points over the UNMODIFIED reference sources.
//
// TEST INFRASTRUCTURE ONLY (parity oracle + the bench's reference arm).
// Built by oracle/build_ref.sh together with
//   /root/reference/proj/src/{tensor_ops,selection,attention,token_coverage}.cpp
// (compiled where they lie, never copied) into oracle/_ref/libtsa_ref.so.
// Each function only marshals raw f32 arrays into the reference's own types
// (tsa::HeadTensors, tsa::HeadScores, ...) and calls the reference function.
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "tsa/attention.hpp"
#include "tsa/model.hpp"
#include "tsa/tensor_ops.hpp"
#include "tsa/token_coverage.hpp"

using namespace tsa;

namespace {

thread_local std::string g_err;

Matrix to_mat(const float* p, int rows, int cols) {
    Matrix m(rows, cols);
    if (rows * cols) std::memcpy(m.data(), p, sizeof(float) * size_t(rows) * size_t(cols));
    return m;
}

void from_mat(const Matrix& m, float* out) {
    if (m.size()) std::memcpy(out, m.data(), sizeof(float) * size_t(m.size()));
}

HeadTensors make_heads(const float* q, const float* k, const float* v, int H, int Hkv, int L,
                       int d) {
    HeadTensors ht;
    for (int h = 0; h < H; ++h) ht.q.push_back(to_mat(q + size_t(h) * L * d, L, d));
    for (int h = 0; h < Hkv; ++h) {
        ht.k.push_back(to_mat(k + size_t(h) * L * d, L, d));
        if (v) ht.v.push_back(to_mat(v + size_t(h) * L * d, L, d));
        else ht.v.push_back(Matrix::Zero(L, d));
    }
    return ht;
}

template <typename F>
int guarded(F f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

template <typename F>
void parallel_heads(int n, int n_threads, F f) {
    n_threads = std::max(1, std::min(n_threads, n));
    if (n_threads == 1) {
        for (int i = 0; i < n; ++i) f(i);
        return;
    }
    std::atomic<int> next{0};
    std::vector<std::thread> th;
    std::vector<std::exception_ptr> errs(static_cast<size_t>(n_threads));
    for (int t = 0; t < n_threads; ++t)
        th.emplace_back([&, t] {
            try {
                for (int i = next++; i < n; i = next++) f(i);
            } catch (...) {
                errs[size_t(t)] = std::current_exception();
            }
        });
    for (auto& x : th) x.join();
    for (auto& e : errs)
        if (e) std::rethrow_exception(e);
}

}  // namespace

extern "C" {

const char* tsa_ref_last_error(void) { return g_err.c_str(); }

// token_coverage.hpp:32.  Single-threaded: exactly the reference call.
int tsa_ref_score_tokens(const float* q, const float* k, int H, int Hkv, int L, int d, int last_q,
                         int kernel, float* s_out) {
    return guarded([&] {
        const HeadTensors ht = make_heads(q, k, nullptr, H, Hkv, L, d);
        from_mat(score_tokens(ht, last_q, kernel).s, s_out);
    });
}

// Head-parallel form: each worker calls the reference score_tokens on a
// one-head HeadTensors (same per-head arithmetic, token_coverage.cpp:24-49).
int tsa_ref_score_tokens_mt(const float* q, const float* k, int H, int Hkv, int L, int d,
                            int last_q, int kernel, float* s_out, int n_threads) {
    return guarded([&] {
        if (H % Hkv != 0) throw std::invalid_argument("score_tokens: H % Hkv != 0");
        const int g = H / Hkv;
        parallel_heads(H, n_threads, [&](int h) {
            HeadTensors one;
            one.q.push_back(to_mat(q + size_t(h) * L * d, L, d));
            one.k.push_back(to_mat(k + size_t(h / g) * L * d, L, d));
            one.v.push_back(Matrix::Zero(1, d));
            const HeadScores hs = score_tokens(one, last_q, kernel);
            from_mat(hs.s, s_out + size_t(h) * L);
        });
    });
}

int tsa_ref_aggregate_scores(const float* s, int H, int L, float* sl_out) {
    return guarded([&] {
        HeadScores hs;
        hs.s = to_mat(s, H, L);
        from_mat(Matrix(aggregate_scores(hs).s.transpose()), sl_out);
    });
}

int tsa_ref_coverage_budget(const float* sl, int L, double tau, int min_keep, int* k_keep) {
    return guarded([&] {
        LayerScores ls;
        ls.s = Vector(to_mat(sl, L, 1));
        *k_keep = coverage_budget(ls, tau, min_keep);
    });
}

int tsa_ref_fixed_budget(int L, double s, int min_keep, int* k_keep) {
    return guarded([&] { *k_keep = fixed_budget(L, s, min_keep); });
}

int tsa_ref_select_tokens(const float* s, int H, int L, int k_keep, const int* forced, int n_forced,
                          int* idx_out) {
    return guarded([&] {
        HeadScores hs;
        hs.s = to_mat(s, H, L);
        const IndexList f(forced, forced + n_forced);
        const TokenSelection sel = select_tokens(hs, k_keep, f);
        for (int h = 0; h < H; ++h)
            std::copy(sel.indices[size_t(h)].begin(), sel.indices[size_t(h)].end(),
                      idx_out + size_t(h) * size_t(k_keep));
    });
}

int tsa_ref_dense_causal_attention(const float* q, const float* k, const float* v, int n, int d,
                                   float* out) {
    return guarded([&] {
        from_mat(dense_causal_attention(to_mat(q, n, d), to_mat(k, n, d), to_mat(v, n, d)), out);
    });
}

int tsa_ref_masked_sparse_oracle(const float* q, const float* k, const float* v, int n, int d,
                                 const int* s, int ns, float* out) {
    return guarded([&] {
        const IndexList idx(s, s + ns);
        from_mat(masked_sparse_oracle(to_mat(q, n, d), to_mat(k, n, d), to_mat(v, n, d), idx), out);
    });
}

// attention.hpp:44-45, default inner.  out is [H x L x d].
int tsa_ref_token_sparse_attention(const float* q, const float* k, const float* v, int H, int Hkv,
                                   int L, int d, const int* idx, int k_keep, const int* forced,
                                   int n_forced, float* out) {
    return guarded([&] {
        const HeadTensors ht = make_heads(q, k, v, H, Hkv, L, d);
        TokenSelection sel;
        sel.k_keep = k_keep;
        sel.forced.assign(forced, forced + n_forced);
        for (int h = 0; h < H; ++h)
            sel.indices.emplace_back(idx + size_t(h) * k_keep, idx + size_t(h + 1) * k_keep);
        const std::vector<Matrix> o = token_sparse_attention(ht, sel);
        for (int h = 0; h < H; ++h) from_mat(o[size_t(h)], out + size_t(h) * L * d);
    });
}

// Bounded sample of token_sparse_attention for large L (bench reference arm):
// for head h, the reference's gather_rows and dense_causal_attention on the
// first m compressed rows.  Causality makes those rows exactly the first m
// rows of the full call (attention.cpp:25-40 is row-local); the reference
// materialises m x m scores, so its cost grows as m^2.
int tsa_ref_tsa_head_prefix(const float* q, const float* k, const float* v, int H, int Hkv, int L,
                            int d, const int* idx, int k_keep, int h, int m, float* out) {
    return guarded([&] {
        const int kv = h / (H / Hkv);
        const IndexList s(idx + size_t(h) * k_keep, idx + size_t(h) * k_keep + m);
        const Matrix qc = gather_rows(to_mat(q + size_t(h) * L * d, L, d), s);
        const Matrix kc = gather_rows(to_mat(k + size_t(kv) * L * d, L, d), s);
        const Matrix vc = gather_rows(to_mat(v + size_t(kv) * L * d, L, d), s);
        from_mat(dense_causal_attention(qc, kc, vc), out);
    });
}

// ---- attention-branch producer (model.cpp:81-158): rms_norm, apply_rope,
// project_qkv.  Row-major f32 arrays; positions are 0..rows-1 (project_qkv).
int tsa_ref_rms_norm(const float* x, const float* gain, int rows, int cols, float eps, float* out) {
    return guarded([&] {
        Vector g(cols);
        for (int j = 0; j < cols; ++j) g(j) = gain[j];
        from_mat(rms_norm(to_mat(x, rows, cols), g, eps), out);
    });
}

int tsa_ref_apply_rope(const float* x, int rows, int cols, float theta, float* out) {
    return guarded([&] {
        IndexList pos(static_cast<size_t>(rows));
        for (int i = 0; i < rows; ++i) pos[size_t(i)] = i;
        from_mat(apply_rope(to_mat(x, rows, cols), pos, theta), out);
    });
}

// q_out [H x L x d], k_out / v_out [Hkv x L x d]; wq [D x H*d], wk / wv [D x Hkv*d].
int tsa_ref_project_qkv(const float* x_norm, const float* wq, const float* wk, const float* wv,
                        int L, int D, int H, int Hkv, int d, float theta, float* q_out,
                        float* k_out, float* v_out) {
    return guarded([&] {
        ModelConfig cfg;
        cfg.n_heads = H;
        cfg.n_kv_heads = Hkv;
        cfg.d_head = d;
        cfg.d_model = D;
        cfg.rope_theta = theta;
        LayerWeights w;
        w.wq = to_mat(wq, D, H * d);
        w.wk = to_mat(wk, D, Hkv * d);
        w.wv = to_mat(wv, D, Hkv * d);
        const HeadTensors ht = project_qkv(to_mat(x_norm, L, D), w, cfg);
        for (int h = 0; h < H; ++h) from_mat(ht.q[size_t(h)], q_out + size_t(h) * L * d);
        for (int h = 0; h < Hkv; ++h) {
            from_mat(ht.k[size_t(h)], k_out + size_t(h) * L * d);
            from_mat(ht.v[size_t(h)], v_out + size_t(h) * L * d);
        }
    });
}

}  // extern "C"

// ---- drift calibration (drift.cpp:14-65) ----
#include "tsa/drift.hpp"
extern "C" {
// hidden: n_mats row-major [rows x cols] f32 matrices back to back; R_out [n_mats - 1].
int tsa_ref_compute_drift(const float* hidden, int n_mats, int rows, int cols, double epsilon,
                          double* R_out) {
    return guarded([&] {
        std::vector<Matrix> h;
        for (int i = 0; i < n_mats; ++i) h.push_back(to_mat(hidden + size_t(i) * rows * cols, rows, cols));
        const std::vector<double> R = compute_drift(h, epsilon);
        std::copy(R.begin(), R.end(), R_out);
    });
}

int tsa_ref_select_sparse_layers(const double* R, int n, double delta, double* R_hat_out,
                                 int* layers_out, int* n_layers) {
    return guarded([&] {
        const DriftProfile p = select_sparse_layers(std::vector<double>(R, R + n), delta);
        std::copy(p.R_hat.begin(), p.R_hat.end(), R_hat_out);
        std::copy(p.sparse_layers.begin(), p.sparse_layers.end(), layers_out);
        *n_layers = static_cast<int>(p.sparse_layers.size());
    });
}
}  // extern "C"

// ---- FLOP model (flops.cpp:12-51) ----
#include "tsa/flops.hpp"
extern "C" {
// k_keep[i] < 0 marks a dense layer (nullopt); out: dense, sparse, overhead, attn_ratio,
// est_speedup, avg_map_sparsity.
int tsa_ref_estimate_flops(int seq_len, int d_head, int n_heads, const int* k_keep, int n_layers,
                           int last_q, int kernel, double* out) {
    return guarded([&] {
        std::vector<std::optional<int>> b;
        for (int i = 0; i < n_layers; ++i)
            b.push_back(k_keep[i] < 0 ? std::nullopt : std::optional<int>(k_keep[i]));
        const FlopReport r = estimate_flops(seq_len, d_head, n_heads, b, last_q, kernel);
        out[0] = r.dense_flops;
        out[1] = r.sparse_flops;
        out[2] = r.overhead_flops;
        out[3] = r.attn_ratio;
        out[4] = r.est_speedup;
        out[5] = r.avg_map_sparsity;
    });
}
}  // extern "C"
