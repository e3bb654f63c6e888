// K1 FAST: token-importance scoring on the tensor cores (bf16, d = 128).
//
// score_tokens (token_coverage.cpp:16-50) computes, per query head, softmax
// rows of the trailing lq queries against all L keys and sums them by column.
// Per KV group the g*lq tail rows form M-tiles of 128 rows (hpt = 128/lq heads
// per tile, lq in {32, 64, 96, 128}), and the key axis is split into chunks so
// the grid fills the GPU (2 CTAs per SM):
//
//   pass 1 (score_pass1): S = Q_tail K_j^T on tcgen05 (TMEM lane = query
//     row), per-row online max / sum-exp over the chunk's key tiles -> partials
//   pass 2 (score_pass2): the transposed product S^T = K_j Q_tail^T (TMEM lane =
//     key), so each thread owns one key column: it combines the per-row
//     partials (broadcast from shared memory), exponentiates its column and
//     sums it per head in registers -- no cross-thread reduction -> colraw[h, j]
//   pool: the shared edge-clamped pool kernel over colraw.
//
// Warp roles as in attend_sm100.cu: warp 0 TMA (Q tail once, K ring), warp 1
// MMA (S double-buffered in TMEM), warps 2..5 the per-thread math.
// Deterministic: every sum has a fixed order.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>

#include "common.cuh"
#include "sm100.cuh"

namespace tsa {

int make_bf16_map_2d(CUtensorMap* m, const void* base, uint64_t rows, uint32_t box_rows);

namespace {

using namespace tsa_dev;

constexpr int SF_BM = 128, SF_BN = 128, SF_HD = 128, SF_NS = 2;
constexpr int SF_TILE = SF_BM * SF_HD * 2;
constexpr int SF_HALF = SF_TILE / 2;
constexpr int SF_MAX_CHUNKS = 512;

struct __align__(1024) ScoreSmem {
    uint8_t q[SF_TILE];
    uint8_t k[SF_NS][SF_TILE];
    alignas(16) float row_off[SF_BM];  // pass 2: -(m_r + log2 l_r), -inf for padding rows
    uint64_t q_full;
    uint64_t k_full[SF_NS];
    uint64_t k_empty[SF_NS];
    uint64_t s_full[2];
    uint64_t s_free[2];
    uint32_t tmem_base;
};

struct TileGeom {
    int mtile, chunk, kv, h_first, n_heads_tile, kt0, nt;
};

__device__ __forceinline__ TileGeom tile_geom(int L, int group, int hpt, int tiles_per_kv,
                                              int n_chunks) {
    TileGeom g;
    g.mtile = blockIdx.y;
    g.chunk = blockIdx.x;
    g.kv = g.mtile / tiles_per_kv;
    const int sub_t = g.mtile % tiles_per_kv;
    g.h_first = g.kv * group + sub_t * hpt;
    g.n_heads_tile = min(hpt, group - sub_t * hpt);
    const int n_ktiles = (L + SF_BN - 1) / SF_BN;
    const int per = (n_ktiles + n_chunks - 1) / n_chunks;
    g.kt0 = g.chunk * per;
    g.nt = min(n_ktiles, g.kt0 + per) - g.kt0;
    return g;
}

// Shared prologue: barriers + TMEM; warp 0 streams Q tail and K tiles; warp 1
// issues S = Q K^T (kTransposed: S^T = K Q^T) into a double-buffered TMEM tile.
template <bool kTransposed>
__device__ __forceinline__ void producer_roles(ScoreSmem& sm, const CUtensorMap* tm_q,
                                               const CUtensorMap* tm_k, const TileGeom& g, int L,
                                               int lq, uint32_t warp, uint32_t lane) {
    const uint32_t t_s[2] = {sm.tmem_base, sm.tmem_base + 128};
    if (warp == 0) {
        if (lane == 0) {
            for (int i = 0; i < g.n_heads_tile; ++i) {
                const int row = (g.h_first + i) * L + (L - lq);
                tma_load_2d(sm.q + i * lq * 128, tm_q, &sm.q_full, 0, row);
                tma_load_2d(sm.q + SF_HALF + i * lq * 128, tm_q, &sm.q_full, 64, row);
            }
            mbar_arrive_expect_tx(&sm.q_full, g.n_heads_tile * lq * SF_HD * 2);
            for (int j = 0; j < g.nt; ++j) {
                const int st = j % SF_NS;
                if (j >= SF_NS) mbar_wait(&sm.k_empty[st], ((j / SF_NS) - 1) & 1);
                const int r = g.kv * L + (g.kt0 + j) * SF_BN;
                tma_load_2d(sm.k[st], tm_k, &sm.k_full[st], 0, r);
                tma_load_2d(sm.k[st] + SF_HALF, tm_k, &sm.k_full[st], 64, r);
                mbar_arrive_expect_tx(&sm.k_full[st], SF_TILE);
            }
        }
    } else if (warp == 1) {
        // converged warp, elected issue: the MMAs go out back to back from
        // uniform registers (see attend_sm100.cu)
        const uint32_t L1 = elect_one() ? 1u : 0u;
        const uint32_t idesc = idesc_bf16_f32(SF_BM, SF_BN, 0, 0);
        const uint32_t q_base = smem_u32(sm.q);
        mbar_wait(&sm.q_full, 0);
        for (int j = 0; j < g.nt; ++j) {
            const int st = j % SF_NS, b = j & 1;
            mbar_wait(&sm.k_full[st], (j / SF_NS) & 1);
            if (j >= 2) mbar_wait(&sm.s_free[b], ((j - 2) >> 1) & 1);
            tc_fence_after();
            const uint32_t k_base = smem_u32(sm.k[st]);
#pragma unroll
            for (int kk = 0; kk < SF_HD / 16; ++kk) {
                const uint32_t off = (kk >> 2) * SF_HALF + (kk & 3) * 32;
                const uint64_t da = sdesc_kmajor_sw128((kTransposed ? k_base : q_base) + off);
                const uint64_t db = sdesc_kmajor_sw128((kTransposed ? q_base : k_base) + off);
                mma_bf16_ss_p(t_s[b], da, db, idesc, kk > 0 ? 1u : 0u, L1);
            }
            mma_commit_p(&sm.s_full[b], L1);
            mma_commit_p(&sm.k_empty[st], L1);
        }
    }
}

__device__ __forceinline__ void setup(ScoreSmem& sm, uint32_t warp) {
    if (threadIdx.x == 0) {
        mbar_init(&sm.q_full, 1);
        for (int s = 0; s < SF_NS; ++s) {
            mbar_init(&sm.k_full[s], 1);
            mbar_init(&sm.k_empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&sm.s_full[b], 1);
            mbar_init(&sm.s_free[b], 128);
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(&sm.tmem_base, 256);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
}

__device__ __forceinline__ void load_row128(uint32_t taddr, uint32_t (&r)[128]) {
    tmem_ld32_at<0>(taddr, r);
    tmem_ld32_at<32>(taddr + 32, r);
    tmem_ld32_at<64>(taddr + 64, r);
    tmem_ld32_at<96>(taddr + 96, r);
    tmem_wait_ld();
}

// ---------------------------------------------------------------- pass 1
__global__ void __launch_bounds__(192, 2)
score_pass1(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
            int L, int lq, int group, int hpt, int tiles_per_kv, int n_chunks, float scale_log2,
            float2* __restrict__ partial) {
    extern __shared__ uint8_t smem_raw[];
    ScoreSmem& sm = *reinterpret_cast<ScoreSmem*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const TileGeom g = tile_geom(L, group, hpt, tiles_per_kv, n_chunks);
    const uint32_t warp = warp_id_uniform(), lane = lane_id();
    float2* part = partial + ((size_t)g.mtile * n_chunks + g.chunk) * SF_BM;
    if (g.nt <= 0) {
        if (threadIdx.x < SF_BM) part[threadIdx.x] = make_float2(-INFINITY, 0.0f);
        return;
    }
    setup(sm, warp);
    producer_roles<false>(sm, &tm_q, &tm_k, g, L, lq, warp, lane);
    if (warp >= 2) {
        const uint32_t sub = warp & 3;
        const int row = (int)(sub * 32 + lane);  // tile row = TMEM lane
        const int r = row % lq;
        const int limit = L - lq + r;            // last key this row may see
        const uint32_t lane_off = (sub * 32) << 16;
        float m_run = -INFINITY, l_run = 0.0f;
        for (int j = 0; j < g.nt; ++j) {
            const int b = j & 1;
            const int key0 = (g.kt0 + j) * SF_BN;
            mbar_wait(&sm.s_full[b], (j >> 1) & 1);
            tc_fence_after();
            uint32_t x[SF_BN];
            load_row128(sm.tmem_base + b * 128 + lane_off, x);
            tc_fence_before();
            mbar_arrive(&sm.s_free[b]);
            if (key0 + SF_BN - 1 > limit) {
#pragma unroll
                for (int c = 0; c < SF_BN; ++c)
                    if (key0 + c > limit) x[c] = __float_as_uint(-INFINITY);
            }
            // row max: 8 partial maxima seeded by columns 0..15, then 7 x 16 columns
            float pm[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) pm[e] = fmaxf(__uint_as_float(x[e]), __uint_as_float(x[8 + e]));
#pragma unroll
            for (int c = 16; c < SF_BN; c += 16)
#pragma unroll
                for (int e = 0; e < 8; ++e)
                    pm[e] = max3f(pm[e], __uint_as_float(x[c + e]), __uint_as_float(x[c + 8 + e]));
            const float tmax = max3f(max3f(pm[0], pm[1], pm[2]), max3f(pm[3], pm[4], pm[5]),
                                     fmaxf(pm[6], pm[7])) * scale_log2;
            const float m_new = fmaxf(m_run, tmax);
            if (m_new != -INFINITY) {
                // packed f32x2 scale (FFMA2) and partial sums (FADD2)
                const uint64_t sc2 = f2(scale_log2, scale_log2), nm2 = f2(-m_new, -m_new);
                uint64_t ps[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
                for (int c = 0; c < SF_BN; c += 2) {
                    float y0, y1;
                    f2_split(fma2(f2(__uint_as_float(x[c]), __uint_as_float(x[c + 1])), sc2, nm2), y0,
                             y1);
                    // every 4th pair on the FMA pipe (the kernel is MUFU-bound)
                    const uint64_t e = ((c >> 1) & 3) == 3
                                           ? ex2_poly2(f2(fmaxf(y0, -127.0f), fmaxf(y1, -127.0f)))
                                           : f2(ex2_approx(y0), ex2_approx(y1));
                    ps[(c >> 1) & 3] = add2(ps[(c >> 1) & 3], e);
                }
                float s0, s1;
                f2_split(add2(add2(ps[0], ps[1]), add2(ps[2], ps[3])), s0, s1);
                l_run = l_run * ex2_approx(m_run - m_new) + (s0 + s1);
                m_run = m_new;
            }
        }
        part[row] = make_float2(m_run, l_run);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(sm.tmem_base, 256);
}

// ---------------------------------------------------------------- pass 2
template <int LQ>
__global__ void __launch_bounds__(192, 2)
score_pass2(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
            int L, int group, int hpt, int tiles_per_kv, int n_chunks, float scale_log2,
            const float2* __restrict__ partial, float* __restrict__ colraw) {
    constexpr int HPT_MAX = 128 / LQ;
    extern __shared__ uint8_t smem_raw[];
    ScoreSmem& sm = *reinterpret_cast<ScoreSmem*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const TileGeom g = tile_geom(L, group, hpt, tiles_per_kv, n_chunks);
    const uint32_t warp = warp_id_uniform(), lane = lane_id();
    if (g.nt <= 0) return;
    // combine the chunk partials of every query row (thread t -> row t)
    if (threadIdx.x < SF_BM) {
        const int row = threadIdx.x;
        const float2* part = partial + (size_t)g.mtile * n_chunks * SF_BM + row;
        float M = -INFINITY;
        for (int c = 0; c < n_chunks; ++c) M = fmaxf(M, part[(size_t)c * SF_BM].x);
        float Ls = 0.0f;
        for (int c = 0; c < n_chunks; ++c) {
            const float2 p = part[(size_t)c * SF_BM];
            if (p.y > 0.0f) Ls += p.y * ex2_approx(p.x - M);
        }
        const bool valid = row / LQ < g.n_heads_tile && Ls > 0.0f;
        // p = 2^(x scale - m) / l = 2^(x scale - (m + log2 l)): the normaliser
        // folds into the exponent offset (one FFMA per element, no multiply)
        sm.row_off[row] = valid ? -(M + __log2f(Ls)) : -INFINITY;
    }
    setup(sm, warp);  // includes __syncthreads: row stats visible
    producer_roles<true>(sm, &tm_q, &tm_k, g, L, LQ, warp, lane);
    if (warp >= 2) {
        const uint32_t sub = warp & 3;
        const int t = (int)(sub * 32 + lane);  // key within the tile = TMEM lane
        const uint32_t lane_off = (sub * 32) << 16;
        for (int j = 0; j < g.nt; ++j) {
            const int b = j & 1;
            const int key = (g.kt0 + j) * SF_BN + t;
            mbar_wait(&sm.s_full[b], (j >> 1) & 1);
            tc_fence_after();
            uint32_t x[SF_BN];  // x[c] = q_row_c . k_key (column c = tail row of the tile)
            load_row128(sm.tmem_base + b * 128 + lane_off, x);
            tc_fence_before();
            mbar_arrive(&sm.s_free[b]);
            // rows r may see this key iff key <= L - lq + r  <=>  r >= key - (L - lq);
            // all but the last tile(s) are visible to every row (warp-uniform test)
            const int r_first = key - (L - LQ);
            const bool tile_full = (g.kt0 + j) * SF_BN + SF_BN - 1 <= L - LQ;
            const uint64_t sc2 = f2(scale_log2, scale_log2);
            float acc[HPT_MAX];
#pragma unroll
            for (int i = 0; i < HPT_MAX; ++i) {
                uint64_t a01 = 0ull, a23 = 0ull;
#pragma unroll
                for (int rr = 0; rr < LQ; rr += 4) {
                    const int c = i * LQ + rr;
                    const float4 off = *reinterpret_cast<const float4*>(&sm.row_off[c]);
                    float y0, y1, y2, y3;
                    f2_split(fma2(f2(__uint_as_float(x[c]), __uint_as_float(x[c + 1])), sc2,
                                  f2(off.x, off.y)), y0, y1);
                    f2_split(fma2(f2(__uint_as_float(x[c + 2]), __uint_as_float(x[c + 3])), sc2,
                                  f2(off.z, off.w)), y2, y3);
                    float p0, p1, p2, p3;
                    if ((rr & 12) == 12) {  // a quarter of the pairs on the FMA pipe
                        f2_split(ex2_poly2(f2(fmaxf(y0, -127.0f), fmaxf(y1, -127.0f))), p0, p1);
                        p2 = ex2_approx(y2);
                        p3 = ex2_approx(y3);
                    } else {
                        p0 = ex2_approx(y0);
                        p1 = ex2_approx(y1);
                        p2 = ex2_approx(y2);
                        p3 = ex2_approx(y3);
                    }
                    if (!tile_full) {
                        p0 = rr + 0 >= r_first ? p0 : 0.0f;
                        p1 = rr + 1 >= r_first ? p1 : 0.0f;
                        p2 = rr + 2 >= r_first ? p2 : 0.0f;
                        p3 = rr + 3 >= r_first ? p3 : 0.0f;
                    }
                    a01 = add2(a01, f2(p0, p1));
                    a23 = add2(a23, f2(p2, p3));
                }
                float s0, s1;
                f2_split(add2(a01, a23), s0, s1);
                acc[i] = s0 + s1;
            }
            if (key < L) {
#pragma unroll
                for (int i = 0; i < HPT_MAX; ++i)
                    if (i < g.n_heads_tile) colraw[(size_t)(g.h_first + i) * L + key] = acc[i];
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(sm.tmem_base, 256);
}

template <int LQ>
int launch_pass2(dim3 grid, int smem, cudaStream_t st, const CUtensorMap& mq, const CUtensorMap& mk,
                 int L, int g, int hpt, int tpk, int n_chunks, float sl2, const float2* partial,
                 float* colraw) {
    if (int rc = ensure_smem_attr(reinterpret_cast<const void*>(score_pass2<LQ>), smem)) return rc;
    score_pass2<LQ><<<grid, 192, smem, st>>>(mq, mk, L, g, hpt, tpk, n_chunks, sl2, partial, colraw);
    TSA_LAUNCH_CHECK("score_fast_pass2");
    return 0;
}

}  // namespace

bool score_fast_available() { return true; }

namespace {
struct FastGeom {
    int lq, g, hpt, tiles_per_kv, kv_begin, n_kv, mtiles, n_ktiles;
};
FastGeom fast_geom(const tsa_desc& d) {
    FastGeom f;
    f.lq = lq_of(d);
    f.g = d.n_heads / d.n_kv_heads;
    f.hpt = std::min(128 / f.lq, f.g);
    f.tiles_per_kv = (f.g + f.hpt - 1) / f.hpt;
    f.kv_begin = d.head_begin / f.g;
    f.n_kv = d.head_end / f.g - f.kv_begin;
    f.mtiles = f.n_kv * f.tiles_per_kv;
    f.n_ktiles = (d.seq_len + SF_BN - 1) / SF_BN;
    return f;
}
}  // namespace

// Row partials of pass 1: mtiles x n_chunks x 128 float2, n_chunks <= the
// key-tile count and SF_MAX_CHUNKS -- sized for the whole layer (every shard
// fits), independent of the device's SM count.
size_t score_fast_rowstat_bytes(const tsa_desc& d) {
    tsa_desc all = d;
    all.head_begin = 0;
    all.head_end = d.n_heads;
    if (d.last_q < 1 || d.n_kv_heads < 1) return 0;
    const FastGeom f = fast_geom(all);
    if (f.lq > 128) return 0;
    return (size_t)f.mtiles * std::min(f.n_ktiles, SF_MAX_CHUNKS) * SF_BM * sizeof(float2);
}

bool score_fast_supported(const tsa_desc& d) {
    const int lq = lq_of(d);
    return d.dtype == TSA_BF16 && d.d_head == SF_HD && lq % 32 == 0 && lq <= 128;
}

int launch_score_fast(const tsa_desc& d, const void* q, const void* k, const OutReplicas& s,
                      float* colraw,
                      float* partial_ws, cudaStream_t st) {
    if (!score_fast_supported(d))
        return invalid("score_tokens: FAST scoring needs bf16, d_head 128 and last_q (clamped to "
                       "L) a multiple of 32 up to 128");
    const int L = d.seq_len;
    const FastGeom f = fast_geom(d);
    const int lq = f.lq, g = f.g, hpt = f.hpt, tiles_per_kv = f.tiles_per_kv;
    const int kv_begin = f.kv_begin, n_kv = f.n_kv, mtiles = f.mtiles, n_ktiles = f.n_ktiles;
    const int n_chunks =
        std::max(1, std::min({n_ktiles, SF_MAX_CHUNKS, (4 * num_sms() + mtiles - 1) / mtiles}));
    // the workspace holds every chunk partial (score_fast_rowstat_bytes)
    if ((size_t)mtiles * n_chunks * SF_BM * sizeof(float2) > score_fast_rowstat_bytes(d))
        return invalid("score_fast: row-partial workspace too small");
    // shard-local views: heads [head_begin, head_end) start at kv_begin
    const size_t eb = 2;
    const uint8_t* qb = static_cast<const uint8_t*>(q) + (size_t)kv_begin * g * L * SF_HD * eb;
    const uint8_t* kb = static_cast<const uint8_t*>(k) + (size_t)kv_begin * L * SF_HD * eb;
    CUtensorMap mq, mk;
    int rc;
    if ((rc = make_bf16_map_2d(&mq, qb, (uint64_t)n_kv * g * L, (uint32_t)lq))) return rc;
    if ((rc = make_bf16_map_2d(&mk, kb, (uint64_t)n_kv * L, 128))) return rc;
    const int smem = (int)sizeof(ScoreSmem) + 1024;
    if ((rc = ensure_smem_attr(reinterpret_cast<const void*>(score_pass1), smem))) return rc;
    const float sl2 = (1.0f / sqrtf((float)SF_HD)) * 1.4426950408889634f;
    float2* partial = reinterpret_cast<float2*>(partial_ws);
    float* colraw_local = colraw + (size_t)d.head_begin * L;  // indexed by local head
    dim3 grid(n_chunks, mtiles);
    score_pass1<<<grid, 192, smem, st>>>(mq, mk, L, lq, g, hpt, tiles_per_kv, n_chunks, sl2, partial);
    TSA_LAUNCH_CHECK("score_fast_pass1");
    switch (lq) {
        case 32: rc = launch_pass2<32>(grid, smem, st, mq, mk, L, g, hpt, tiles_per_kv, n_chunks, sl2, partial, colraw_local); break;
        case 64: rc = launch_pass2<64>(grid, smem, st, mq, mk, L, g, hpt, tiles_per_kv, n_chunks, sl2, partial, colraw_local); break;
        case 96: rc = launch_pass2<96>(grid, smem, st, mq, mk, L, g, hpt, tiles_per_kv, n_chunks, sl2, partial, colraw_local); break;
        default: rc = launch_pass2<128>(grid, smem, st, mq, mk, L, g, hpt, tiles_per_kv, n_chunks, sl2, partial, colraw_local); break;
    }
    if (rc) return rc;
    // pool over the raw column sums (one "row" per head)
    tsa_desc pd = d;
    pd.last_q = 1;
    return launch_colsum_pool(pd, colraw, s, st);
}

}  // namespace tsa
