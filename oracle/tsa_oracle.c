/*
 * tsa_oracle.c -- CPU restatement of the reference Token Sparse Attention path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * path in paper_2602_03216_b200/.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  The product
 * never links or calls it.
 *
 * Every routine restates /root/reference/proj (file:line cited per function)
 * with the same f32 operation order: the reference is built with
 * -ffp-contract=off (proj/CMakeLists.txt:14-16), so there is no FMA anywhere
 * and each a*b+c below is a separate multiply and add (this file must be
 * compiled with -ffp-contract=off as well, see oracle/Makefile).
 *
 * Parity pinning: tests/test_oracle.py checks this file bit-for-bit against
 * the reference sources compiled here (oracle/_ref, oracle/build_ref.sh) and
 * against the reference's inline known-answer tests.
 *
 * Layout contract (reference HeadTensors, attention.hpp:16-25): q is H blocks
 * of [L x d] row-major f32, k and v are Hkv blocks; kv_head(h) = h / (H/Hkv).
 */
#include <errno.h>
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define EXPORT __attribute__((visibility("default")))

static __thread char g_err[512];

EXPORT const char* tsa_oracle_last_error(void) { return g_err; }

static int fail(const char* fmt, long a, long b, long c) {
    snprintf(g_err, sizeof g_err, fmt, a, b, c);
    return 1;
}

/* ------------------------------------------------------------------ RNG */
/* std::mt19937_64 (bit-specified by the standard) and tsa::Rng
 * (random.hpp:16-33): uniform() = (gen() >> 40) * 2^-24. */
typedef struct {
    uint64_t mt[312];
    int idx;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
}

static uint64_t mt64_next(mt64* g) {
    if (g->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (g->mt[i] & 0xFFFFFFFF80000000ULL) | (g->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
        }
        g->idx = 0;
    }
    uint64_t y = g->mt[g->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= (y >> 43);
    return y;
}

/* bench.cpp:31-36 */
EXPORT uint64_t tsa_oracle_mix_seed(uint64_t seed, uint64_t stream) {
    uint64_t z = seed + 0x9E3779B97F4A7C15ULL * (stream + 1);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* Opaque generator handle so Python can reproduce random_matrix streams
 * (random.hpp:36-44: row-major fill, lo + (hi - lo) * uniform()). */
EXPORT void* tsa_oracle_rng_new(uint64_t seed) {
    mt64* g = (mt64*)malloc(sizeof(mt64));
    if (g) mt64_seed(g, seed);
    return g;
}
EXPORT void tsa_oracle_rng_free(void* g) { free(g); }
EXPORT void tsa_oracle_rng_fill(void* g, int64_t n, float scale, float* out) {
    const float lo = -scale, hi = scale;
    for (int64_t i = 0; i < n; ++i) {
        const float u = (float)(mt64_next((mt64*)g) >> 40) * 0x1p-24f;
        out[i] = lo + (hi - lo) * u;
    }
}
EXPORT uint64_t tsa_oracle_rng_raw(void* g) { return mt64_next((mt64*)g); }

/* -------------------------------------------------------------- helpers */
/* tensor_ops.cpp:12-25: C(i,:) += A(i,p) * B(p,:), p ascending, no FMA.
 * Here B is given transposed (bt = [n x d] = K) so the call site reads like
 * matmul(Q, K^T); the per-element order is identical. */
static void row_logits(const float* qrow, const float* kt /* [d x n] */, int n, int d,
                       int n_used, float* out) {
    for (int j = 0; j < n_used; ++j) out[j] = 0.0f;
    for (int p = 0; p < d; ++p) {
        const float a = qrow[p];
        const float* b = kt + (size_t)p * n;
        for (int j = 0; j < n_used; ++j) {
            const float t = a * b[j];
            out[j] = out[j] + t;
        }
    }
    (void)n;
}

static float* transpose(const float* m, int rows, int cols) {
    float* t = (float*)malloc(sizeof(float) * (size_t)rows * cols);
    if (!t) return NULL;
    for (int i = 0; i < rows; ++i)
        for (int j = 0; j < cols; ++j) t[(size_t)j * rows + i] = m[(size_t)i * cols + j];
    return t;
}

/* Masked softmax of one row whose allowed entries are the prefix [0, n_allowed)
 * (tensor_ops.cpp:40-71): max over unmasked (first unmasked seeds it,
 * std::max after), e = expf(x - mx), sequential f32 sum, then divide.
 * Masked entries are exactly +0. */
static void softmax_prefix(float* row, int n_allowed, int n_total) {
    float mx = row[0];
    for (int j = 1; j < n_allowed; ++j) mx = (mx < row[j]) ? row[j] : mx;
    float sum = 0.0f;
    for (int j = 0; j < n_allowed; ++j) {
        const float e = expf(row[j] - mx);
        row[j] = e;
        sum = sum + e;
    }
    for (int j = 0; j < n_allowed; ++j) row[j] = row[j] / sum;
    for (int j = n_allowed; j < n_total; ++j) row[j] = 0.0f;
}

/* Eigen's vectorised sum of a short segment: with SSE2 packets of 4 floats
 * and 16-byte aligned storage, Eigen's redux peels to the first aligned
 * index, sums one packet with predux = (a0+a2)+(a1+a3), then adds the head
 * and tail scalars in order (Eigen Redux.h, LinearVectorizedTraversal).
 * `base` is the absolute index of seg[0] in the 16-byte-aligned vector. */
static float eigen_segment_sum(const float* seg, int n, int base) {
    int a = (4 - (base & 3)) & 3;
    if (a > n) a = n;
    const int aligned_size = ((n - a) / 4) * 4;
    if (aligned_size == 0) {
        float r = seg[0];
        for (int i = 1; i < n; ++i) r = r + seg[i];
        return r;
    }
    /* aligned_size is 4 for n <= 7 (kernel <= 7); general case: 2-packet accumulate. */
    float p0[4], p1[4];
    for (int l = 0; l < 4; ++l) p0[l] = seg[a + l];
    const int aligned_end = a + aligned_size;
    if (aligned_size > 4) {
        const int aligned_size2 = ((n - a) / 8) * 8;
        const int aligned_end2 = a + aligned_size2;
        for (int l = 0; l < 4; ++l) p1[l] = seg[a + 4 + l];
        for (int i = a + 8; i < aligned_end2; i += 8) {
            for (int l = 0; l < 4; ++l) p0[l] = p0[l] + seg[i + l];
            for (int l = 0; l < 4; ++l) p1[l] = p1[l] + seg[i + 4 + l];
        }
        for (int l = 0; l < 4; ++l) p0[l] = p0[l] + p1[l];
        if (aligned_end > aligned_end2)
            for (int l = 0; l < 4; ++l) p0[l] = p0[l] + seg[aligned_end2 + l];
    }
    float r = (p0[0] + p0[2]) + (p0[1] + p0[3]);
    for (int i = 0; i < a; ++i) r = r + seg[i];
    for (int i = aligned_end; i < n; ++i) r = r + seg[i];
    return r;
}

/* tensor_ops.cpp:114-129: same-length edge-clamped mean pool. */
static int avg_pool_1d(const float* v, int n, int kernel, float* out) {
    if (kernel < 1 || kernel % 2 == 0)
        return fail("avg_pool_1d: kernel must be odd and positive, got %ld", kernel, 0, 0);
    if (kernel == 1) {
        memcpy(out, v, sizeof(float) * (size_t)n);
        return 0;
    }
    const int h = kernel / 2;
    for (int t = 0; t < n; ++t) {
        const int lo = t - h > 0 ? t - h : 0;
        const int hi = t + h < n - 1 ? t + h : n - 1;
        const int cnt = hi - lo + 1;
        out[t] = eigen_segment_sum(v + lo, cnt, lo) / (float)cnt;
    }
    return 0;
}

EXPORT int tsa_oracle_avg_pool_1d(const float* v, int n, int kernel, float* out) {
    return avg_pool_1d(v, n, kernel, out);
}

/* ------------------------------------------------------ threading helper */
typedef struct {
    void (*fn)(void* ctx, int item);
    void* ctx;
    int n_items;
    int next;
    pthread_mutex_t mu;
} pool_t;

static void* pool_worker(void* arg) {
    pool_t* p = (pool_t*)arg;
    for (;;) {
        pthread_mutex_lock(&p->mu);
        const int it = p->next++;
        pthread_mutex_unlock(&p->mu);
        if (it >= p->n_items) break;
        p->fn(p->ctx, it);
    }
    return NULL;
}

static void parallel_for(int n_items, int n_threads, void (*fn)(void*, int), void* ctx) {
    if (n_threads <= 1 || n_items <= 1) {
        for (int i = 0; i < n_items; ++i) fn(ctx, i);
        return;
    }
    if (n_threads > n_items) n_threads = n_items;
    pool_t p = {fn, ctx, n_items, 0, PTHREAD_MUTEX_INITIALIZER};
    pthread_t th[256];
    if (n_threads > 256) n_threads = 256;
    for (int t = 0; t < n_threads; ++t) pthread_create(&th[t], NULL, pool_worker, &p);
    for (int t = 0; t < n_threads; ++t) pthread_join(th[t], NULL);
}

/* ------------------------------------------------------------ scoring */
typedef struct {
    const float *q, *k;
    int H, Hkv, L, d, lq, kernel;
    float* s;
    int err;
} score_ctx;

/* token_coverage.cpp:16-50 for one query head. */
static void score_one_head(void* vctx, int h) {
    score_ctx* c = (score_ctx*)vctx;
    const int L = c->L, d = c->d, lq = c->lq;
    const int kv = h / (c->H / c->Hkv); /* attention.hpp:24 */
    const float* q = c->q + (size_t)h * L * d;
    const float* k = c->k + (size_t)kv * L * d;
    const float inv_sqrt_d = 1.0f / sqrtf((float)d); /* :31 */
    float* kt = transpose(k, L, d);                   /* Matrix(k.transpose()) :32 */
    float* row = (float*)malloc(sizeof(float) * (size_t)L);
    float* col = (float*)calloc((size_t)L, sizeof(float)); /* Vector::Zero :43 */
    if (!kt || !row || !col) {
        c->err = 1;
        free(kt), free(row), free(col);
        return;
    }
    for (int r = 0; r < lq; ++r) {
        /* matmul(q.bottomRows(lq), K^T) row r, then *= inv_sqrt_d (:32-33) */
        /* entries past the causal limit are masked to exact 0 below, so only
         * the allowed prefix of the logits row is computed */
        const float* qrow = q + (size_t)(L - lq + r) * d;
        const int allowed = L - lq + r + 1;
        row_logits(qrow, kt, L, d, allowed, row);
        for (int j = 0; j < allowed; ++j) row[j] = row[j] * inv_sqrt_d;
        /* mask j <= L - lq + r (:36-41), masked softmax (:42) */
        softmax_prefix(row, L - lq + r + 1, L);
        /* col_sums += proxy.row(r)^T (:44-46) */
        for (int j = 0; j < L; ++j) col[j] = col[j] + row[j];
    }
    if (avg_pool_1d(col, L, c->kernel, c->s + (size_t)h * L)) c->err = 2; /* :47 */
    free(kt), free(row), free(col);
}

EXPORT int tsa_oracle_score_tokens(const float* q, const float* k, int H, int Hkv, int L, int d,
                                   int last_q, int kernel, float* s_out, int n_threads) {
    if (last_q < 1) return fail("score_tokens: last_q must be positive, got %ld", last_q, 0, 0);
    if (H < 1 || Hkv < 1 || H % Hkv != 0)
        return fail("score_tokens: %ld query heads not divisible by %ld KV heads", H, Hkv, 0);
    if (L < 1 || d < 1) return fail("score_tokens: bad shape L=%ld d=%ld", L, d, 0);
    if (kernel < 1 || kernel % 2 == 0)
        return fail("avg_pool_1d: kernel must be odd and positive, got %ld", kernel, 0, 0);
    score_ctx c = {q, k, H, Hkv, L, d, last_q < L ? last_q : L, kernel, s_out, 0};
    parallel_for(H, n_threads, score_one_head, &c);
    if (c.err) return fail("score_tokens: internal error %ld", c.err, 0, 0);
    return 0;
}

/* token_coverage.cpp:52-66 */
EXPORT int tsa_oracle_aggregate_scores(const float* s, int H, int L, float* sl_out) {
    float* sum = (float*)calloc((size_t)L, sizeof(float));
    if (!sum) return fail("aggregate_scores: out of memory", 0, 0, 0);
    for (int h = 0; h < H; ++h)
        for (int t = 0; t < L; ++t) sum[t] = sum[t] + s[(size_t)h * L + t];
    float total = 0.0f;
    for (int t = 0; t < L; ++t) total = total + sum[t];
    if (!(total > 0.0f)) {
        free(sum);
        return fail("aggregate_scores: all scores are zero, cannot normalize", 0, 0, 0);
    }
    for (int t = 0; t < L; ++t) sl_out[t] = sum[t] / total;
    free(sum);
    return 0;
}

/* Stable ascending merge sort of indices by key (std::stable_sort semantics). */
typedef struct {
    const float* key;
    int desc;
} sort_ctx;

static int before(const sort_ctx* c, int a, int b) {
    return c->desc ? (c->key[a] > c->key[b]) : (c->key[a] < c->key[b]);
}

static void stable_sort_idx(int* idx, int n, const sort_ctx* c) {
    int* tmp = (int*)malloc(sizeof(int) * (size_t)(n > 0 ? n : 1));
    for (int w = 1; w < n; w *= 2) {
        for (int lo = 0; lo < n; lo += 2 * w) {
            int mid = lo + w < n ? lo + w : n, hi = lo + 2 * w < n ? lo + 2 * w : n;
            int i = lo, j = mid, o = lo;
            while (i < mid && j < hi) tmp[o++] = before(c, idx[j], idx[i]) ? idx[j++] : idx[i++];
            while (i < mid) tmp[o++] = idx[i++];
            while (j < hi) tmp[o++] = idx[j++];
        }
        memcpy(idx, tmp, sizeof(int) * (size_t)n);
    }
    free(tmp);
}

/* token_coverage.cpp:68-96.  *prefix_at (optional) receives the double
 * prefix at the crossing and *prefix_prev the one before it, so tests can
 * state how close a budget boundary is to tau. */
EXPORT int tsa_oracle_coverage_budget_ex(const float* sl, int L, double tau, int min_keep,
                                         int* k_keep, double* prefix_prev, double* prefix_at) {
    if (tau < 0.0 || tau > 1.0) {
        snprintf(g_err, sizeof g_err, "coverage_budget: tau %f outside [0, 1]", tau);
        return 1;
    }
    if (min_keep < 1 || min_keep > L)
        return fail("coverage_budget: min_keep %ld outside [1, %ld]", min_keep, L, 0);
    int* order = (int*)malloc(sizeof(int) * (size_t)L);
    for (int i = 0; i < L; ++i) order[i] = i;
    sort_ctx c = {sl, 0};
    stable_sort_idx(order, L, &c);
    int k_sparse = L;
    double prefix = 0.0, prev = 0.0;
    if (prefix >= tau) {
        k_sparse = 0;
    } else {
        for (int k = 1; k <= L; ++k) {
            prev = prefix;
            prefix += (double)sl[order[k - 1]];
            if (prefix >= tau) {
                k_sparse = k;
                break;
            }
        }
    }
    free(order);
    if (prefix_prev) *prefix_prev = prev;
    if (prefix_at) *prefix_at = prefix;
    *k_keep = (L - k_sparse) > min_keep ? (L - k_sparse) : min_keep;
    return 0;
}

EXPORT int tsa_oracle_coverage_budget(const float* sl, int L, double tau, int min_keep,
                                      int* k_keep) {
    return tsa_oracle_coverage_budget_ex(sl, L, tau, min_keep, k_keep, NULL, NULL);
}

/* token_coverage.cpp:98-109 */
EXPORT int tsa_oracle_fixed_budget(int L, double s, int min_keep, int* k_keep) {
    if (s < 0.0 || s >= 1.0) {
        snprintf(g_err, sizeof g_err, "fixed_budget: sparsity ratio %f outside [0, 1)", s);
        return 1;
    }
    if (min_keep < 1 || min_keep > L)
        return fail("fixed_budget: min_keep %ld outside [1, %ld]", min_keep, L, 0);
    const int k = (int)lround((1.0 - s) * L);
    *k_keep = k > min_keep ? k : min_keep;
    return 0;
}

/* model.cpp:74-79: kFinalToken -> {L-1}; kRecentWindow -> [max(0, L-last_q), L). */
EXPORT int tsa_oracle_forced_set(int L, int policy, int last_q, int* out) {
    if (policy == 0) {
        out[0] = L - 1;
        return 1;
    }
    int n = 0;
    for (int t = (L - last_q > 0 ? L - last_q : 0); t < L; ++t) out[n++] = t;
    return n;
}

static int cmp_int(const void* a, const void* b) {
    const int x = *(const int*)a, y = *(const int*)b;
    return (x > y) - (x < y);
}

typedef struct {
    const float* s;
    int L, k_keep, nf;
    const int* f;
    const char* is_forced;
    const int* pool;
    int n_pool;
    int* idx_out;
} select_ctx;

static void select_one_head(void* vctx, int h) {
    select_ctx* c = (select_ctx*)vctx;
    int* ranked = (int*)malloc(sizeof(int) * (size_t)(c->n_pool > 0 ? c->n_pool : 1));
    memcpy(ranked, c->pool, sizeof(int) * (size_t)c->n_pool);
    sort_ctx sc = {c->s + (size_t)h * c->L, 1};
    stable_sort_idx(ranked, c->n_pool, &sc); /* :141-145, ties -> lower index */
    int* out = c->idx_out + (size_t)h * c->k_keep;
    int n = 0;
    for (int i = 0; i < c->nf; ++i) out[n++] = c->f[i];
    for (int i = 0; i < c->k_keep - c->nf; ++i) out[n++] = ranked[i];
    qsort(out, (size_t)n, sizeof(int), cmp_int); /* :146-148 */
    free(ranked);
}

/* token_coverage.cpp:111-152.  idx_out is [H x k_keep]. */
EXPORT int tsa_oracle_select_tokens(const float* s, int H, int L, int k_keep, const int* forced,
                                    int n_forced, int* idx_out, int n_threads) {
    int* f = (int*)malloc(sizeof(int) * (size_t)(n_forced > 0 ? n_forced : 1));
    memcpy(f, forced, sizeof(int) * (size_t)n_forced);
    qsort(f, (size_t)n_forced, sizeof(int), cmp_int);
    int nf = 0;
    for (int i = 0; i < n_forced; ++i)
        if (nf == 0 || f[nf - 1] != f[i]) f[nf++] = f[i];
    for (int i = 0; i < nf; ++i)
        if (f[i] < 0 || f[i] >= L) {
            int t = f[i];
            free(f);
            return fail("select_tokens: forced index %ld out of range [0, %ld)", t, L, 0);
        }
    const int min_keep = nf > 1 ? nf : 1;
    if (k_keep < min_keep || k_keep > L) {
        free(f);
        return fail("select_tokens: k_keep %ld outside [%ld, %ld]", k_keep, min_keep, L);
    }
    char* is_forced = (char*)calloc((size_t)L, 1);
    for (int i = 0; i < nf; ++i) is_forced[f[i]] = 1;
    int* pool = (int*)malloc(sizeof(int) * (size_t)L);
    int n_pool = 0;
    for (int t = 0; t < L; ++t)
        if (!is_forced[t]) pool[n_pool++] = t;
    select_ctx c = {s, L, k_keep, nf, f, is_forced, pool, n_pool, idx_out};
    parallel_for(H, n_threads, select_one_head, &c);
    free(pool), free(is_forced), free(f);
    return 0;
}

/* ---------------------------------------------------------- attention */
/* attention.cpp:25-40, rows [r0, r1) only.  Every output row depends only on
 * its own score row, so computing a row range is bit-identical to the full
 * call; P.V skips the p > i terms, which are exact +0 products that cannot
 * change an accumulator that started at +0 (round-to-nearest never yields
 * -0 from +0 + (+-0)). */
static void dense_rows(const float* q, const float* kt, const float* v, int n, int d, int r0, int r1,
                       float* out /* [(r1-r0) x d] */, float* row) {
    const float inv_sqrt_d = 1.0f / sqrtf((float)d);
    for (int i = r0; i < r1; ++i) {
        row_logits(q + (size_t)i * d, kt, n, d, i + 1, row);
        for (int j = 0; j <= i; ++j) row[j] = row[j] * inv_sqrt_d;
        softmax_prefix(row, i + 1, i + 1);
        float* o = out + (size_t)(i - r0) * d;
        for (int c = 0; c < d; ++c) o[c] = 0.0f;
        for (int p = 0; p <= i; ++p) {
            const float a = row[p];
            const float* vr = v + (size_t)p * d;
            for (int c = 0; c < d; ++c) {
                const float t = a * vr[c];
                o[c] = o[c] + t;
            }
        }
    }
}

EXPORT int tsa_oracle_dense_causal_attention_rows(const float* q, const float* k, const float* v,
                                                  int n, int d, int r0, int r1, float* out) {
    if (n < 1 || d < 1 || r0 < 0 || r1 > n || r0 > r1)
        return fail("dense_causal_attention: bad shape n=%ld d=%ld rows=%ld", n, d, r1 - r0);
    float* kt = transpose(k, n, d);
    float* row = (float*)malloc(sizeof(float) * (size_t)n);
    dense_rows(q, kt, v, n, d, r0, r1, out, row);
    free(kt), free(row);
    return 0;
}

EXPORT int tsa_oracle_dense_causal_attention(const float* q, const float* k, const float* v, int n,
                                             int d, float* out) {
    return tsa_oracle_dense_causal_attention_rows(q, k, v, n, d, 0, n, out);
}

/* attention.cpp:42-72 for one head. */
EXPORT int tsa_oracle_masked_sparse_oracle(const float* q, const float* k, const float* v, int n,
                                           int d, const int* s, int ns, float* out) {
    char* in_s = (char*)calloc((size_t)n, 1);
    for (int r = 0; r < ns; ++r) {
        if (s[r] < 0 || s[r] >= n) {
            free(in_s);
            return fail("masked_sparse_oracle: index %ld out of range [0, %ld)", s[r], n, 0);
        }
        if (r > 0 && s[r] <= s[r - 1]) {
            free(in_s);
            return fail("masked_sparse_oracle: indices must be strictly ascending", 0, 0, 0);
        }
        in_s[s[r]] = 1;
    }
    const float inv_sqrt_d = 1.0f / sqrtf((float)d);
    float* kt = transpose(k, n, d);
    float* row = (float*)malloc(sizeof(float) * (size_t)n);
    float* p = (float*)malloc(sizeof(float) * (size_t)n);
    memset(out, 0, sizeof(float) * (size_t)n * d);
    for (int i = 0; i < n; ++i) {
        if (!in_s[i]) continue;
        row_logits(q + (size_t)i * d, kt, n, d, n, row);
        /* allowed: j in S and j <= i; masked softmax over that set (:63-70) */
        float mx = 0.0f;
        int any = 0;
        for (int j = 0; j <= i; ++j) {
            if (!in_s[j]) continue;
            const float x = row[j] * inv_sqrt_d;
            mx = any ? ((mx < x) ? x : mx) : x;
            any = 1;
        }
        float sum = 0.0f;
        for (int j = 0; j < n; ++j) {
            p[j] = 0.0f;
            if (j > i || !in_s[j]) continue;
            const float e = expf(row[j] * inv_sqrt_d - mx);
            p[j] = e;
            sum = sum + e;
        }
        for (int j = 0; j <= i; ++j)
            if (in_s[j]) p[j] = p[j] / sum;
        float* o = out + (size_t)i * d;
        for (int jj = 0; jj < n; ++jj) {
            const float a = p[jj];
            const float* vr = v + (size_t)jj * d;
            for (int c = 0; c < d; ++c) {
                const float t = a * vr[c];
                o[c] = o[c] + t;
            }
        }
    }
    free(kt), free(row), free(p), free(in_s);
    return 0;
}

typedef struct {
    const float *q, *k, *v;
    int H, Hkv, L, d, k_keep;
    const int* idx;
    float* out;
    /* row sampling: per head only compressed rows [r0, r1) are produced */
    int r0, r1;
    int head_stride; /* process heads h = item * head_stride (sampling) */
} tsa_ctx;

/* attention.cpp:74-99 for one head: gather -> dense_causal_attention -> scatter. */
static void tsa_one_head(void* vctx, int item) {
    tsa_ctx* c = (tsa_ctx*)vctx;
    const int h = item * c->head_stride;
    const int L = c->L, d = c->d, k = c->k_keep;
    const int kv = h / (c->H / c->Hkv);
    const int* s = c->idx + (size_t)h * k;
    float* qc = (float*)malloc(sizeof(float) * (size_t)k * d);
    float* kc = (float*)malloc(sizeof(float) * (size_t)k * d);
    float* vc = (float*)malloc(sizeof(float) * (size_t)k * d);
    for (int r = 0; r < k; ++r) { /* gather_rows, tensor_ops.cpp:92-99 */
        memcpy(qc + (size_t)r * d, c->q + ((size_t)h * L + s[r]) * d, sizeof(float) * d);
        memcpy(kc + (size_t)r * d, c->k + ((size_t)kv * L + s[r]) * d, sizeof(float) * d);
        memcpy(vc + (size_t)r * d, c->v + ((size_t)kv * L + s[r]) * d, sizeof(float) * d);
    }
    const int r0 = c->r0, r1 = c->r1 < k ? c->r1 : k;
    float* oc = (float*)malloc(sizeof(float) * (size_t)(r1 > r0 ? r1 - r0 : 1) * d);
    float* kt = transpose(kc, k, d);
    float* row = (float*)malloc(sizeof(float) * (size_t)k);
    dense_rows(qc, kt, vc, k, d, r0, r1, oc, row);
    /* scatter_rows, tensor_ops.cpp:101-112: zero-init, then place rows */
    float* o = c->out + (size_t)h * L * d;
    memset(o, 0, sizeof(float) * (size_t)L * d);
    for (int r = r0; r < r1; ++r)
        memcpy(o + (size_t)s[r] * d, oc + (size_t)(r - r0) * d, sizeof(float) * d);
    free(qc), free(kc), free(vc), free(oc), free(kt), free(row);
}

static int check_selection(const int* idx, int H, int L, int k_keep) {
    if (k_keep < 1 || k_keep > L) return fail("validate: k_keep %ld outside [1, %ld]", k_keep, L, 0);
    for (int h = 0; h < H; ++h) {
        const int* s = idx + (size_t)h * k_keep;
        for (int r = 0; r < k_keep; ++r) {
            if (s[r] < 0 || s[r] >= L)
                return fail("validate: head %ld index %ld out of range [0, %ld)", h, s[r], L);
            if (r > 0 && s[r] <= s[r - 1])
                return fail("validate: head %ld indices not strictly ascending at position %ld", h,
                            r, 0);
        }
    }
    return 0;
}

/* Full operator: out is [H x L x d]. */
EXPORT int tsa_oracle_token_sparse_attention(const float* q, const float* k, const float* v, int H,
                                             int Hkv, int L, int d, const int* idx, int k_keep,
                                             float* out, int n_threads) {
    if (H < 1 || Hkv < 1 || H % Hkv != 0)
        return fail("token_sparse_attention: %ld query heads not divisible by %ld KV heads", H, Hkv,
                    0);
    if (check_selection(idx, H, L, k_keep)) return 1;
    tsa_ctx c = {q, k, v, H, Hkv, L, d, k_keep, idx, out, 0, k_keep, 1};
    parallel_for(H, n_threads, tsa_one_head, &c);
    return 0;
}

/* Sampled variant for large L (bench cpu_baseline / parity at full size):
 * heads 0, head_stride, 2*head_stride, ...; compressed rows [r0, r1) per head.
 * Produces exactly the rows the full call would produce for those heads. */
EXPORT int tsa_oracle_token_sparse_attention_sampled(const float* q, const float* k, const float* v,
                                                     int H, int Hkv, int L, int d, const int* idx,
                                                     int k_keep, int head_stride, int r0, int r1,
                                                     float* out, int n_threads) {
    if (H < 1 || Hkv < 1 || H % Hkv != 0 || head_stride < 1)
        return fail("token_sparse_attention: bad heads %ld/%ld stride %ld", H, Hkv, head_stride);
    if (check_selection(idx, H, L, k_keep)) return 1;
    tsa_ctx c = {q, k, v, H, Hkv, L, d, k_keep, idx, out, r0, r1, head_stride};
    parallel_for((H + head_stride - 1) / head_stride, n_threads, tsa_one_head, &c);
    return 0;
}

/* ---------------------------------------------------------------------------
 * Attention-branch producer (callers upstream of the path).
 * rms_norm      model.cpp:81-94   ss = sum_j x^2 (f32, j ascending), inv = 1 / sqrt(ss / D + eps),
 *                                 out = (x * inv) * gain
 * apply_rope    model.cpp:96-123  pairs (2i, 2i+1) rotated by pos * theta^(-2i/d): angle in
 *                                 double, (float)cos / (float)sin, x0 c - x1 s, x0 s + x1 c (f32)
 * project_qkv   model.cpp:139-158 matmul (tensor_ops.cpp:12-25, p ascending, no FMA), split
 *                                 into heads, RoPE on q and k at positions 0..L-1
 */
EXPORT int tsa_oracle_rms_norm(const float* x, const float* gain, int rows, int cols, float eps,
                               float* out) {
    if (rows < 0 || cols < 1) return fail("rms_norm: bad shape %ld x %ld", rows, cols, 0);
    for (int i = 0; i < rows; ++i) {
        const float* xr = x + (size_t)i * cols;
        float ss = 0.0f;
        for (int j = 0; j < cols; ++j) ss += xr[j] * xr[j];
        const float inv = 1.0f / sqrtf(ss / (float)cols + eps);
        for (int j = 0; j < cols; ++j) out[(size_t)i * cols + j] = xr[j] * inv * gain[j];
    }
    return 0;
}

EXPORT int tsa_oracle_apply_rope(const float* x, int rows, int cols, float theta, float* out) {
    if (cols % 2 != 0) return fail("apply_rope: odd head dimension %ld", cols, 0, 0);
    const int half = cols / 2;
    for (int r = 0; r < rows; ++r) {
        for (int i = 0; i < half; ++i) {
            const double freq = pow((double)theta, -2.0 * (double)i / (double)cols);
            const double angle = (double)r * freq;
            const float c = (float)cos(angle), s = (float)sin(angle);
            const float x0 = x[(size_t)r * cols + 2 * i], x1 = x[(size_t)r * cols + 2 * i + 1];
            out[(size_t)r * cols + 2 * i] = x0 * c - x1 * s;
            out[(size_t)r * cols + 2 * i + 1] = x0 * s + x1 * c;
        }
    }
    return 0;
}

/* C[n x m] = A[n x k] B[k x m], reference order: C(i, :) += A(i, p) B(p, :), p ascending. */
static void matmul_ref(const float* A, const float* B, int n, int k, int m, float* Cm) {
    for (size_t i = 0; i < (size_t)n * m; ++i) Cm[i] = 0.0f;
    for (int i = 0; i < n; ++i)
        for (int p = 0; p < k; ++p) {
            const float a = A[(size_t)i * k + p];
            const float* b = B + (size_t)p * m;
            float* c = Cm + (size_t)i * m;
            for (int j = 0; j < m; ++j) c[j] += a * b[j];
        }
}

/* q_out [H x L x d]; k_out / v_out [Hkv x L x d]; wq [D x H d], wk / wv [D x Hkv d]. */
EXPORT int tsa_oracle_project_qkv(const float* x_norm, const float* wq, const float* wk,
                                  const float* wv, int L, int D, int H, int Hkv, int d,
                                  float theta, float* q_out, float* k_out, float* v_out) {
    if (H < 1 || Hkv < 1 || d < 2 || d % 2) return fail("project_qkv: bad heads %ld/%ld d %ld", H, Hkv, d);
    const int widths[3] = {H * d, Hkv * d, Hkv * d};
    const float* ws[3] = {wq, wk, wv};
    float* outs[3] = {q_out, k_out, v_out};
    const int nh[3] = {H, Hkv, Hkv};
    float* proj = (float*)malloc(sizeof(float) * (size_t)L * H * d);
    float* head = (float*)malloc(sizeof(float) * (size_t)L * d);
    if (!proj || !head) {
        free(proj);
        free(head);
        return fail("project_qkv: out of memory", 0, 0, 0);
    }
    for (int t = 0; t < 3; ++t) {
        matmul_ref(x_norm, ws[t], L, D, widths[t], proj);
        for (int h = 0; h < nh[t]; ++h) {
            for (int r = 0; r < L; ++r)
                memcpy(head + (size_t)r * d, proj + (size_t)r * widths[t] + (size_t)h * d,
                       sizeof(float) * d);
            float* dst = outs[t] + (size_t)h * L * d;
            if (t < 2) tsa_oracle_apply_rope(head, L, d, theta, dst);
            else memcpy(dst, head, sizeof(float) * (size_t)L * d);
        }
    }
    free(proj);
    free(head);
    return 0;
}

/* ---------------------------------------------------------------------------
 * Drift calibration (drift.cpp:14-65): R[l] = mean_t |h[l+1][t] - h[l][t]|_2 /
 * (|h[l][t]|_2 + eps), sums in double with j and t ascending; normalized ranks
 * R_hat[l] = #{k : R[k] <= R[l]} / n and the sparse set {l : R_hat[l] <= delta}.
 */
EXPORT int tsa_oracle_compute_drift(const float* hidden, int n_mats, int rows, int cols,
                                    double epsilon, double* R_out) {
    if (n_mats < 2) return fail("compute_drift: need at least 2 hidden-state matrices, got %ld",
                                n_mats, 0, 0);
    if (!(epsilon > 0)) return fail("compute_drift: epsilon must be positive", 0, 0, 0);
    for (int l = 0; l + 1 < n_mats; ++l) {
        const float* a = hidden + (size_t)l * rows * cols;
        const float* b = a + (size_t)rows * cols;
        double acc = 0.0;
        for (int t = 0; t < rows; ++t) {
            double num = 0.0, den = 0.0;
            for (int j = 0; j < cols; ++j) {
                const double d = (double)b[(size_t)t * cols + j] - a[(size_t)t * cols + j];
                num += d * d;
                den += (double)a[(size_t)t * cols + j] * a[(size_t)t * cols + j];
            }
            acc += sqrt(num) / (sqrt(den) + epsilon);
        }
        R_out[l] = acc / (double)rows;
    }
    return 0;
}

EXPORT int tsa_oracle_select_sparse_layers(const double* R, int n, double delta, double* R_hat,
                                           int* layers, int* n_layers) {
    if (n < 1) return fail("select_sparse_layers: empty drift vector", 0, 0, 0);
    int m = 0;
    for (int l = 0; l < n; ++l) {
        int count = 0;
        for (int k = 0; k < n; ++k)
            if (R[k] <= R[l]) ++count;
        R_hat[l] = (double)count / (double)n;
        if (R_hat[l] <= delta) layers[m++] = l;
    }
    *n_layers = m;
    return 0;
}

/* The softmax exponential as the reference evaluates it: std::exp(float) is
 * the host libm's expf (tensor_ops.cpp:62).  Batch form for the GPU parity
 * test of the exact scorer's expf port (tests/test_gpu_exact.py). */
EXPORT void tsa_oracle_expf(const float* x, float* y, int64_t n) {
    for (int64_t i = 0; i < n; ++i) y[i] = expf(x[i]);
}
