// K1 FAST: token-importance scoring on the tensor cores (bf16, d = 128).
//
// score_tokens (token_coverage.cpp:16-50) computes, per query head, softmax
// rows of the trailing lq queries against all L keys and sums them by column.
// Per KV group the g*lq tail rows form M-tiles of 128 rows (hpt = 128/lq heads
// per tile, lq % 32 == 0), and the key axis is split into chunks so the grid
// fills the GPU:
//
//   pass 1 (score_fast_kernel<false>): S = Q_tail K_j^T on tcgen05 (TMEM),
//     per-row online max / sum-exp over the chunk's key tiles -> partials
//   pass 2 (score_fast_kernel<true>):  combine the partials of all chunks,
//     recompute S, P = 2^(x - M) / l, column sums per head by an in-warp
//     butterfly reduce-scatter (lane l ends with columns 4l..4l+3) plus a
//     fixed-order cross-warp sum -> colraw[h, j]  (deterministic)
//   pool: the shared edge-clamped pool kernel over colraw.
//
// Warp roles as in attend_sm100.cu: warp 0 TMA (Q tail once, K ring), warp 1
// MMA (S double-buffered in TMEM), warps 2..5 one query row per thread.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>

#include "common.cuh"
#include "sm100.cuh"

namespace tsa {

int make_bf16_map_2d(CUtensorMap* m, const void* base, uint64_t rows, uint32_t box_rows);

namespace {

using namespace tsa_dev;

constexpr int SF_BM = 128, SF_BN = 128, SF_HD = 128, SF_NS = 3;
constexpr int SF_TILE = SF_BM * SF_HD * 2;
constexpr int SF_HALF = SF_TILE / 2;
constexpr int SF_MAX_CHUNKS = 512;

struct __align__(1024) ScoreSmem {
    uint8_t q[SF_TILE];
    uint8_t k[SF_NS][SF_TILE];
    float red[4][SF_BN];
    uint64_t q_full;
    uint64_t k_full[SF_NS];
    uint64_t k_empty[SF_NS];
    uint64_t s_full[2];
    uint64_t s_free[2];
    uint32_t tmem_base;
};

template <bool kPass2>
__global__ void __launch_bounds__(192, 1)
score_fast_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                  int L, int lq, int group, int hpt, int tiles_per_kv, int n_chunks,
                  float scale_log2, float2* __restrict__ partial, float* __restrict__ colraw) {
    extern __shared__ uint8_t smem_raw[];
    ScoreSmem& sm = *reinterpret_cast<ScoreSmem*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int mtile = blockIdx.y, chunk = blockIdx.x;
    const int kv = mtile / tiles_per_kv, sub_t = mtile % tiles_per_kv;
    const int h_first = kv * group + sub_t * hpt;
    const int n_heads_tile = min(hpt, group - sub_t * hpt);
    const int n_ktiles = (L + SF_BN - 1) / SF_BN;
    const int per = (n_ktiles + n_chunks - 1) / n_chunks;
    const int kt0 = chunk * per, kt1 = min(n_ktiles, kt0 + per);
    const int nt = kt1 - kt0;
    const uint32_t warp = warp_id_uniform(), lane = lane_id();

    if (nt <= 0) {
        if (!kPass2 && threadIdx.x < SF_BM)
            partial[((size_t)mtile * n_chunks + chunk) * SF_BM + threadIdx.x] =
                make_float2(-INFINITY, 0.0f);
        return;
    }
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
    const uint32_t t_s[2] = {sm.tmem_base, sm.tmem_base + 128};

    if (warp == 0) {
        if (lane == 0) {
            for (int i = 0; i < n_heads_tile; ++i) {
                const int row = (h_first + i) * L + (L - lq);
                tma_load_2d(sm.q + i * lq * 128, &tm_q, &sm.q_full, 0, row);
                tma_load_2d(sm.q + SF_HALF + i * lq * 128, &tm_q, &sm.q_full, 64, row);
            }
            mbar_arrive_expect_tx(&sm.q_full, n_heads_tile * lq * SF_HD * 2);
            for (int j = 0; j < nt; ++j) {
                const int st = j % SF_NS;
                if (j >= SF_NS) mbar_wait(&sm.k_empty[st], ((j / SF_NS) - 1) & 1);
                const int r = kv * L + (kt0 + j) * SF_BN;
                tma_load_2d(sm.k[st], &tm_k, &sm.k_full[st], 0, r);
                tma_load_2d(sm.k[st] + SF_HALF, &tm_k, &sm.k_full[st], 64, r);
                mbar_arrive_expect_tx(&sm.k_full[st], SF_TILE);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t idesc = idesc_bf16_f32(SF_BM, SF_BN, 0, 0);
            const uint32_t q_base = smem_u32(sm.q);
            mbar_wait(&sm.q_full, 0);
            for (int j = 0; j < nt; ++j) {
                const int st = j % SF_NS, b = j & 1;
                mbar_wait(&sm.k_full[st], (j / SF_NS) & 1);
                if (j >= 2) mbar_wait(&sm.s_free[b], ((j - 2) >> 1) & 1);
                tc_fence_after();
                const uint32_t k_base = smem_u32(sm.k[st]);
#pragma unroll
                for (int kk = 0; kk < SF_HD / 16; ++kk) {
                    const uint32_t off = (kk >> 2) * SF_HALF + (kk & 3) * 32;
                    mma_bf16_ss(t_s[b], sdesc_kmajor_sw128(q_base + off),
                                sdesc_kmajor_sw128(k_base + off), idesc, kk > 0 ? 1u : 0u);
                }
                mma_commit(&sm.s_full[b]);
                mma_commit(&sm.k_empty[st]);
            }
        }
    } else {
        const uint32_t sub = warp & 3;
        const int row = (int)(sub * 32 + lane);   // tile row
        const int head_i = row / lq;              // head within tile
        const int r = row % lq;                   // tail row index
        const bool valid = head_i < n_heads_tile;
        const int limit = L - lq + r;             // last key this row may see
        const uint32_t lane_off = (sub * 32) << 16;
        float m_run = -INFINITY, l_run = 0.0f, inv_l = 0.0f;
        if (kPass2) {
            float M = -INFINITY;
            for (int c = 0; c < n_chunks; ++c)
                M = fmaxf(M, partial[((size_t)mtile * n_chunks + c) * SF_BM + row].x);
            float Ls = 0.0f;
            for (int c = 0; c < n_chunks; ++c) {
                const float2 p = partial[((size_t)mtile * n_chunks + c) * SF_BM + row];
                if (p.y > 0.0f) Ls += p.y * ex2_approx(p.x - M);
            }
            m_run = M;
            inv_l = Ls > 0.0f ? 1.0f / Ls : 0.0f;
        }
        for (int j = 0; j < nt; ++j) {
            const int b = j & 1;
            const int key0 = (kt0 + j) * SF_BN;
            mbar_wait(&sm.s_full[b], (j >> 1) & 1);
            tc_fence_after();
            float x[SF_BN];
#pragma unroll
            for (int c = 0; c < SF_BN; c += 32) {
                uint32_t rr[32];
                tmem_ld32(t_s[b] + lane_off + c, rr);
                tmem_wait_ld();
#pragma unroll
                for (int e = 0; e < 32; ++e) x[c + e] = __uint_as_float(rr[e]);
            }
            tc_fence_before();
            mbar_arrive(&sm.s_free[b]);
            const bool edge = key0 + SF_BN - 1 > limit;
#pragma unroll
            for (int c = 0; c < SF_BN; ++c) {
                float v = x[c] * scale_log2;
                if (edge && key0 + c > limit) v = -INFINITY;
                x[c] = v;
            }
            if (!kPass2) {
                float tmax = -INFINITY;
#pragma unroll
                for (int c = 0; c < SF_BN; ++c) tmax = fmaxf(tmax, x[c]);
                const float m_new = fmaxf(m_run, tmax);
                if (m_new != -INFINITY) {
                    float s = 0.0f;
#pragma unroll
                    for (int c = 0; c < SF_BN; ++c) s += ex2_approx(x[c] - m_new);
                    l_run = l_run * ex2_approx(m_run - m_new) + s;
                    m_run = m_new;
                }
            } else {
                // P row, then butterfly reduce-scatter across the warp's 32 rows
#pragma unroll
                for (int c = 0; c < SF_BN; ++c)
                    x[c] = valid ? ex2_approx(x[c] - m_run) * inv_l : 0.0f;
#pragma unroll
                for (int step = 0; step < 5; ++step) {
                    const int half = 64 >> step;          // values kept per lane after the step
                    const uint32_t bit = (lane >> (4 - step)) & 1u;
                    const int xmask = 16 >> step;
#pragma unroll
                    for (int i = 0; i < half; ++i) {
                        const float keep = bit ? x[half + i] : x[i];
                        const float send = bit ? x[i] : x[half + i];
                        x[i] = keep + __shfl_xor_sync(0xffffffffu, send, xmask);
                    }
                }
                // lane holds columns 4*lane .. 4*lane+3 of this warp's 32 rows
#pragma unroll
                for (int e = 0; e < 4; ++e) sm.red[sub][4 * lane + e] = x[e];
                named_bar_sync(1, 128);
                const int c = threadIdx.x - 64;  // 0..127 over the softmax warps
                const int key = key0 + c;
                const int warps_per_head = lq / 32;
                for (int i = 0; i < n_heads_tile; ++i) {
                    float acc = 0.0f;
                    for (int w = 0; w < warps_per_head; ++w) acc += sm.red[i * warps_per_head + w][c];
                    if (key < L) colraw[(size_t)(h_first + i) * L + key] = acc;
                }
                named_bar_sync(1, 128);
            }
        }
        if (!kPass2)
            partial[((size_t)mtile * n_chunks + chunk) * SF_BM + row] = make_float2(m_run, l_run);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(sm.tmem_base, 256);
}

}  // namespace

bool score_fast_available() { return true; }

bool score_fast_supported(const tsa_desc& d) {
    const int lq = lq_of(d);
    const int g = d.n_heads / d.n_kv_heads;
    (void)g;
    return d.dtype == TSA_BF16 && d.d_head == SF_HD && lq % 32 == 0 && lq <= 128;
}

int launch_score_fast(const tsa_desc& d, const void* q, const void* k, float* s, float* colraw,
                      float* partial_ws, cudaStream_t st) {
    if (!score_fast_supported(d))
        return invalid("score_tokens: FAST scoring needs bf16, d_head 128 and last_q (clamped to "
                       "L) a multiple of 32 up to 128");
    const int L = d.seq_len, lq = lq_of(d);
    const int g = d.n_heads / d.n_kv_heads;
    const int hpt = std::min(128 / lq, g);
    const int tiles_per_kv = (g + hpt - 1) / hpt;
    const int kv_begin = d.head_begin / g, kv_end = d.head_end / g;
    const int n_kv = kv_end - kv_begin;
    const int mtiles = n_kv * tiles_per_kv;
    const int n_ktiles = (L + SF_BN - 1) / SF_BN;
    const int n_chunks = std::max(1, std::min({n_ktiles, SF_MAX_CHUNKS, (2 * kNumSMs + mtiles - 1) / mtiles}));
    // shard-local views: heads [head_begin, head_end) start at kv_begin
    const size_t eb = 2;
    const uint8_t* qb = static_cast<const uint8_t*>(q) + (size_t)kv_begin * g * L * SF_HD * eb;
    const uint8_t* kb = static_cast<const uint8_t*>(k) + (size_t)kv_begin * L * SF_HD * eb;
    CUtensorMap mq, mk;
    int rc;
    if ((rc = make_bf16_map_2d(&mq, qb, (uint64_t)n_kv * g * L, (uint32_t)lq))) return rc;
    if ((rc = make_bf16_map_2d(&mk, kb, (uint64_t)n_kv * L, 128))) return rc;
    const int smem = (int)sizeof(ScoreSmem) + 1024;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(score_fast_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(score_fast_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        attr = true;
    }
    const float scale_log2 = (1.0f / sqrtf((float)SF_HD)) * 1.4426950408889634f;
    float2* partial = reinterpret_cast<float2*>(partial_ws);
    float* colraw_local = colraw + (size_t)d.head_begin * L;  // indexed by local head below
    dim3 grid(n_chunks, mtiles);
    score_fast_kernel<false><<<grid, 192, smem, st>>>(mq, mk, L, lq, g, hpt, tiles_per_kv, n_chunks,
                                                      scale_log2, partial, colraw_local);
    TSA_LAUNCH_CHECK("score_fast_pass1");
    score_fast_kernel<true><<<grid, 192, smem, st>>>(mq, mk, L, lq, g, hpt, tiles_per_kv, n_chunks,
                                                     scale_log2, partial, colraw_local);
    TSA_LAUNCH_CHECK("score_fast_pass2");
    // pool over the raw column sums (one "row" per head)
    tsa_desc pd = d;
    pd.last_q = 1;
    return launch_colsum_pool(pd, colraw, s, st);
}

}  // namespace tsa
