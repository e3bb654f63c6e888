// K5: causal flash attention on the 5th-generation tensor cores (sm_100a).
//
// dense_causal_attention (attention.cpp:25-40) -- the `inner` kernel the
// reference applies to the compressed Q^/K^/V^ of each head -- for bf16 and
// d = 128.  One CTA owns a PAIR of 128-row query tiles (A = rows 256p..+127,
// B = rows 256p+128..+255) so every K/V tile that lands in shared memory feeds
// four MMAs, and the two softmax warpgroups ping-pong against the tensor core:
//
//   warp 8        TMA producer: Q_A, Q_B once; K_j and V_j through 2-stage rings
//   warp 9        MMA issuer (one thread), FA4-style order
//                   S_A(0) S_B(0) | PV_A(0) S_A(1) PV_B(0) S_B(1) | PV_A(1) S_A(2) ...
//                 so that while softmax(A, j+1) runs, the tensor core executes
//                 PV_B(j) and S_B(j+1), and vice versa
//   warps 0..3    softmax for tile A, warps 4..7 for tile B: thread = query row =
//                 TMEM lane.  Two passes over the S row in TMEM (max, then
//                 exp2 / sum / bf16 pack) keep registers low; P overwrites the
//                 S columns (tcgen05.st) and is consumed by a TS-MMA.  Lazy
//                 rescaling: O is rescaled only when the running max grows by
//                 more than 2^8 (warp-uniform decision, tcgen05.ld/st are
//                 warp-collective).  S(j) completing implies PV(j-1) completed
//                 (tcgen05.commit tracks all prior MMAs), so the rescale needs
//                 no extra barrier.  Epilogue: O / l -> bf16 -> global.
//
// Warps 8..11 drop to 40 registers (setmaxnreg) so the softmax warpgroups can
// hold a full 128-column S row in registers (232 each).
// TMEM (512 columns): S_A [0,128) S_B [128,256) O_A [256,384) O_B [384,512).
// n (rows per head) is read from device memory (k_keep): the grid is sized for
// L, pairs past n exit before allocating anything, heavy pairs go first.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "sm100.cuh"

namespace tsa {
namespace {

using namespace tsa_dev;

constexpr int BM = 128;                   // rows per query tile
constexpr int BN = 128;                   // keys per KV tile
constexpr int HD = 128;                   // head dim
constexpr int NS = 2;                     // K and V ring stages
constexpr int TILE_BYTES = BM * HD * 2;   // 32 KiB = two 64-column SW128 halves
constexpr int HALF_BYTES = TILE_BYTES / 2;
constexpr float kRescaleThreshold = 8.0f; // log2 units
constexpr int kThreads = 384;             // 12 warps: 2 softmax WGs + producer WG

struct __align__(1024) AttnSmem {
    uint8_t q[2][TILE_BYTES];
    uint8_t k[NS][TILE_BYTES];
    uint8_t v[NS][TILE_BYTES];
    uint64_t q_full;
    uint64_t k_full[NS], v_full[NS], k_empty[NS], v_empty[NS];
    uint64_t s_full[2], p_full[2][4], o_done[2];  // p_full[tile][quarter]
    uint32_t tmem_base;
};

// Shared-memory descriptors differ between the K-steps of one operand only in
// the start-address field (bits 0-13, address >> 4), which never carries into
// the LBO field for shared-memory addresses: build the low word once per
// operand base and add the K-step offset, the high word (SBO = 1 KiB, version,
// SW128 layout) is a constant.
__device__ __forceinline__ uint64_t sdesc_from_lo(uint32_t lo) {
    return (static_cast<uint64_t>(0x40004040u) << 32) | lo;
}
__device__ __forceinline__ uint32_t sdesc_lo(uint32_t saddr, uint32_t lbo_bytes) {
    return ((saddr >> 4) & 0x3FFFu) | (((lbo_bytes >> 4) & 0x3FFFu) << 16);
}

__device__ __forceinline__ void issue_s(uint32_t t_s, uint32_t q_base, uint32_t k_base,
                                        uint32_t idesc, uint32_t leader) {
    const uint32_t qlo = sdesc_lo(q_base, 16), klo = sdesc_lo(k_base, 16);
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
        const uint32_t off = ((kk >> 2) * HALF_BYTES + (kk & 3) * 32) >> 4;
        mma_bf16_ss_p(t_s, sdesc_from_lo(qlo + off), sdesc_from_lo(klo + off), idesc,
                      kk > 0 ? 1u : 0u, leader);
    }
}

// O += P[:, 32q .. 32q+31] V[32q .. 32q+31, :] (quarter q of the 128-key tile).
__device__ __forceinline__ void issue_pv_quarter(uint32_t t_o, uint32_t t_p, uint32_t v_base,
                                                 uint32_t idesc, bool accumulate, int q,
                                                 uint32_t leader) {
    const uint32_t vlo = sdesc_lo(v_base, HALF_BYTES);
#pragma unroll
    for (int k2 = 0; k2 < 2; ++k2) {
        const int kk = q * 2 + k2;
        mma_bf16_ts_p(t_o, t_p + kk * 8, sdesc_from_lo(vlo + ((kk * 2048) >> 4)), idesc,
                      (accumulate || kk > 0) ? 1u : 0u, leader);
    }
}

// P = 2^(x*scale - m) for one 128-key S row held in registers: packed f32x2
// scale (FFMA2), the exponential split between MUFU.EX2 and a polynomial on
// the FMA pipe (pairs set in kPolyMask, per 32-key chunk; the diagonal tile,
// which carries the -inf causal mask, uses kPolyMask = 0), 4 packed partial
// row sums, bf16 pack into S columns [0, 64) (tcgen05.st) with P released to
// the MMA warp in four 32-key quarters (p_full[0..3]) so the PV of the first
// keys overlaps the exponentials of the later ones and only a quarter of the
// PV remains after the last exponential (halves: +2 % at 128K,
// profiles/r1/ab_p_quarters.log).
template <uint32_t kPolyMask>
__device__ __forceinline__ void exp_pack_row(const uint32_t (&r)[BN], uint64_t sc2, uint64_t nm2,
                                             uint32_t t_s, uint64_t* p_full, uint64_t (&ps)[4]) {
#pragma unroll
    for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
            uint64_t x = fma2(f2(__uint_as_float(r[c0 + 2 * e]), __uint_as_float(r[c0 + 2 * e + 1])),
                              sc2, nm2);
            float x0, x1, p0, p1;
            f2_split(x, x0, x1);
            if (kPolyMask >> e & 1u) {
                x = ex2_poly2(f2(fmaxf(x0, -127.0f), fmaxf(x1, -127.0f)));
                f2_split(x, p0, p1);
            } else {
                p0 = ex2_approx(x0);
                p1 = ex2_approx(x1);
                x = f2(p0, p1);
            }
            ps[e & 3] = add2(ps[e & 3], x);
            pk[e] = pack_bf16x2(p0, p1);
        }
        // each 32-key quarter is released once the next chunk's exponentials are
        // in registers, so the wait for its TMEM store overlaps that work
        if (c0 > 0) {
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(&p_full[c0 / 32 - 1]);
        }
        tmem_st16(t_s + c0 / 2, pk);
        if (c0 == 96) {
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(&p_full[3]);
        }
    }
}

// Softmax / correction / epilogue for one 128-row query tile (tile 0 = A, 1 = B).
// Output row of compressed row qi: the compressed buffer (row q_row0 + local
// row) or, for the fused path, the original position h*L + idx[h, qi].
template <uint32_t kPolyMask>
__device__ __forceinline__ void softmax_role(AttnSmem& sm, uint32_t tmem, uint32_t warp,
                                             uint32_t lane, int tA, int tB, bool hasB, int n,
                                             int q_row0, float scale_log2,
                                             const OutReplicas& o,
                                             const int32_t* __restrict__ idx_h, size_t out_head_row) {
        const int tile = warp < 4 ? 0 : 1;  // warps 0..3 -> A, 4..7 -> B
    if (tile == 0 || hasB) {
        const int my_t = tile == 0 ? tA : tB;  // query tile index == its diagonal KV tile
        const uint32_t sub = warp & 3;        // TMEM lane sub-partition
        const int row = (int)(sub * 32 + lane);
        const int qi = my_t * BM + row;
        const uint32_t lane_off = (sub * 32) << 16;
        const uint32_t t_s = tmem + (uint32_t)tile * 128 + lane_off;
        const uint32_t t_o = tmem + 256 + (uint32_t)tile * 128 + lane_off;
        float m_run = -INFINITY, l_run = 0.0f;
        for (int j = 0; j <= my_t; ++j) {
            mbar_wait(&sm.s_full[tile], j & 1);
            tc_fence_after();
            // the whole S row in registers: one TMEM pass, one wait
            uint32_t r[BN];
            tmem_ld32_at<0>(t_s + 0, r);
            tmem_ld32_at<32>(t_s + 32, r);
            tmem_ld32_at<64>(t_s + 64, r);
            tmem_ld32_at<96>(t_s + 96, r);
            tmem_wait_ld();
            if (j == my_t) {  // diagonal tile (warp-uniform): causal mask c > qi - j*BN
                const int lim = qi - j * BN;
#pragma unroll
                for (int c = 0; c < BN; ++c)
                    if (c > lim) r[c] = __float_as_uint(-INFINITY);
            }
            // row max: 8 independent partial maxima, 3-input FMNMX3 (columns
            // 0..15 seed them, then 7 steps of 16 columns cover 16..127)
            float pm[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) pm[e] = fmaxf(__uint_as_float(r[e]), __uint_as_float(r[8 + e]));
#pragma unroll
            for (int c = 16; c < BN; c += 16)
#pragma unroll
                for (int e = 0; e < 8; ++e)
                    pm[e] = max3f(pm[e], __uint_as_float(r[c + e]), __uint_as_float(r[c + 8 + e]));
            const float tmax = max3f(max3f(pm[0], pm[1], pm[2]), max3f(pm[3], pm[4], pm[5]),
                                     fmaxf(pm[6], pm[7])) *
                               scale_log2;
            float m_use = m_run;
            bool rescale = false;
            if (tmax > m_run + kRescaleThreshold || m_run == -INFINITY) {
                m_use = tmax;
                rescale = (m_run != -INFINITY);
            }
            if (m_use == -INFINITY) m_use = 0.0f;  // fully masked row (rows >= n)
            if (__any_sync(0xffffffffu, rescale)) {
                // PV(j-1) is complete: S(j) was issued after it (commit semantics)
                const float alpha = rescale ? ex2_approx(m_run - m_use) : 1.0f;
                const uint64_t alpha2 = f2(alpha, alpha);
#pragma unroll
                for (int c0 = 0; c0 < HD; c0 += 32) {
                    uint32_t ro[32];
                    tmem_ld32(t_o + c0, ro);
                    tmem_wait_ld();
#pragma unroll
                    for (int e = 0; e < 32; e += 2) {
                        float a, b;
                        f2_split(fma2(f2(__uint_as_float(ro[e]), __uint_as_float(ro[e + 1])),
                                      alpha2, 0ull),
                                 a, b);
                        ro[e] = __float_as_uint(a);
                        ro[e + 1] = __float_as_uint(b);
                    }
                    tmem_st32(t_o + c0, ro);
                }
                if (rescale) l_run *= alpha;
            }
            m_run = m_use;
            const uint64_t sc2 = f2(scale_log2, scale_log2), nm2 = f2(-m_use, -m_use);
            uint64_t ps[4] = {0ull, 0ull, 0ull, 0ull};
            if (j == my_t)
                exp_pack_row<0u>(r, sc2, nm2, t_s, sm.p_full[tile], ps);
            else
                exp_pack_row<kPolyMask>(r, sc2, nm2, t_s, sm.p_full[tile], ps);
            float l0, l1;
            f2_split(add2(add2(ps[0], ps[1]), add2(ps[2], ps[3])), l0, l1);
            l_run += l0 + l1;
        }
        // epilogue: wait for the last PV, O / l -> bf16 -> global.  o_done is
        // committed after every PV of the tile but waited only here, for phase
        // my_t: a parity wait is exact when the waiter is at most one phase
        // behind, and it is -- this thread consumed S(my_t), whose commit
        // followed PV(my_t - 1), so phases 0..my_t-1 have completed.  (synccheck
        // reports the unwaited phases as "missing wait"; committing only after
        // the last PV silences it but measured +0.9 % on the 128K layer,
        // profiles/r1/ab_odone_single_commit.log.)
        mbar_wait(&sm.o_done[tile], my_t & 1);
        tc_fence_after();
        const float inv_l = 1.0f / l_run;
        size_t out_row = (size_t)q_row0 + tile * BM + row;
        if (idx_h && qi < n) out_row = out_head_row + (size_t)__ldg(idx_h + qi);
        const size_t out_off = out_row * HD;
#pragma unroll
        for (int c0 = 0; c0 < HD; c0 += 32) {
            uint32_t r[32];
            tmem_ld32(t_o + c0, r);
            tmem_wait_ld();
            if (qi < n) {
                uint4 outv[4];
                uint32_t* ow = reinterpret_cast<uint32_t*>(outv);
#pragma unroll
                for (int e = 0; e < 16; ++e)
                    ow[e] = pack_bf16x2(__uint_as_float(r[2 * e]) * inv_l,
                                        __uint_as_float(r[2 * e + 1]) * inv_l);
                // every output replica (multi-GPU: this rank's buffer and the
                // peers' over NVLink -- the head all-gather fused into the epilogue)
#pragma unroll
                for (int i = 0; i < TSA_MAX_REPLICAS; ++i) {
                    if (i >= o.n) break;
                    uint4* d4 = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(o.p[i]) +
                                                         out_off + c0);
#pragma unroll
                    for (int e = 0; e < 4; ++e) d4[e] = outv[e];
                }
            }
        }
        if (o.n > 1) __threadfence_system();  // peers read after a cross-rank barrier
    }
}

// kIndexed: the fused compress -> attend -> decompress path.  Q rows are
// fetched straight from the original [H, L, d] tensor by the selection
// idx[h, r] with TMA tile::gather4 (4 rows per request, SW128 layout identical
// to the tiled load; once per CTA), K/V tiles stream from the compressed
// per-head buffers, and O rows are stored at their original positions.
// (Gathering K/V with gather4 as well costs 128 TMA requests per KV step and
// measured 2.3x slower on B200; see profiles/r1/README.md.)
template <bool kIndexed, uint32_t kPolyMask>
__global__ void __launch_bounds__(kThreads, 1)
attend_sm100_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_kd,
                    const __grid_constant__ CUtensorMap tm_vd, const __grid_constant__ CUtensorMap tm_v3,
                    const __grid_constant__ CUtensorMap tm_vd3, int dense_group,
                    const int32_t* __restrict__ n_dev,
                    int n_const, int kv_group, int rows_per_head, int kv_rows_per_head,
                    int head_begin, float scale_log2, const __grid_constant__ OutReplicas o,
                    const int32_t* __restrict__ idx) {
    extern __shared__ uint8_t smem_raw[];
    AttnSmem& sm = *reinterpret_cast<AttnSmem*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));

    const int h = head_begin + blockIdx.y;
    const int n = n_dev ? *n_dev : n_const;
    const int n_tiles = (n + BM - 1) / BM;
    const int n_pairs = (n_tiles + 1) / 2;
    if ((int)blockIdx.x >= n_pairs) return;
    const int p = n_pairs - 1 - (int)blockIdx.x;  // heaviest pairs first
    const int tA = 2 * p, tB = 2 * p + 1;
    const bool hasB = tB < n_tiles;
    const int nkv = hasB ? tB + 1 : tA + 1;  // KV tiles 0..nkv-1
    const int kvh = h / kv_group;
    const int kv_row0 = kvh * kv_rows_per_head;
    const int q_row0 = h * rows_per_head + tA * BM;

    const uint32_t warp = warp_id_uniform();
    const uint32_t lane = lane_id();

    if (threadIdx.x == 0) {
        mbar_init(&sm.q_full, 1);
        for (int s = 0; s < NS; ++s) {
            mbar_init(&sm.k_full[s], 1);
            mbar_init(&sm.v_full[s], 1);
            mbar_init(&sm.k_empty[s], 1);
            mbar_init(&sm.v_empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&sm.s_full[b], 1);
            for (int qq = 0; qq < 4; ++qq) mbar_init(&sm.p_full[b][qq], 128);
            mbar_init(&sm.o_done[b], 1);
        }
        fence_barrier_init();
    }
    if (warp == 9) tmem_alloc(&sm.tmem_base, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sm.tmem_base;

    if (warp < 8) {
        // ------------------------------------------------------ softmax warps
        asm volatile("setmaxnreg.inc.sync.aligned.u32 232;\n" ::: "memory");
        softmax_role<kPolyMask>(sm, tmem, warp, lane, tA, tB, hasB, n, q_row0, scale_log2, o,
                     kIndexed ? idx + (size_t)h * rows_per_head : nullptr,
                     (size_t)h * rows_per_head);
        tc_fence_before();
        named_bar_arrive(1, 288);  // teardown: 256 softmax threads + the MMA warp
        return;
    }
    // producer warpgroup: hand registers to the softmax warpgroups
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::: "memory");
    if (warp == 8) {
        // ------------------------------------------------------ TMA producer
        if (!kIndexed) {
            if (lane == 0) {
                tma_load_2d(sm.q[0], &tm_q, &sm.q_full, 0, q_row0);
                tma_load_2d(sm.q[0] + HALF_BYTES, &tm_q, &sm.q_full, 64, q_row0);
                if (hasB) {
                    tma_load_2d(sm.q[1], &tm_q, &sm.q_full, 0, q_row0 + BM);
                    tma_load_2d(sm.q[1] + HALF_BYTES, &tm_q, &sm.q_full, 64, q_row0 + BM);
                }
                mbar_arrive_expect_tx(&sm.q_full, hasB ? 2 * TILE_BYTES : TILE_BYTES);
                for (int j = 0; j < nkv; ++j) {
                    const int st = j % NS;
                    const int r = j * BN;
                    if (j >= NS) mbar_wait(&sm.k_empty[st], ((j / NS) - 1) & 1);
                    tma_load_2d(sm.k[st], &tm_k, &sm.k_full[st], 0, kv_row0 + r);
                    tma_load_2d(sm.k[st] + HALF_BYTES, &tm_k, &sm.k_full[st], 64, kv_row0 + r);
                    mbar_arrive_expect_tx(&sm.k_full[st], TILE_BYTES);
                    if (j >= NS) mbar_wait(&sm.v_empty[st], ((j / NS) - 1) & 1);
                    tma_load_2d(sm.v[st], &tm_v, &sm.v_full[st], 0, kv_row0 + r);
                    tma_load_2d(sm.v[st] + HALF_BYTES, &tm_v, &sm.v_full[st], 64, kv_row0 + r);
                    mbar_arrive_expect_tx(&sm.v_full[st], TILE_BYTES);
                }
            }
        } else {
            // whole warp: lane l gathers rows 4l..4l+3 of every 128-row tile
            const int32_t* idx_h = idx + (size_t)h * rows_per_head;
            const int last = __ldg(idx_h + n - 1);  // rows >= n: any finite row (masked / not stored)
            auto rows4 = [&](int r0, int& a0, int& a1, int& a2, int& a3) {
                a0 = r0 + 0 < n ? __ldg(idx_h + r0 + 0) : last;
                a1 = r0 + 1 < n ? __ldg(idx_h + r0 + 1) : last;
                a2 = r0 + 2 < n ? __ldg(idx_h + r0 + 2) : last;
                a3 = r0 + 3 < n ? __ldg(idx_h + r0 + 3) : last;
            };
            const int q_base_row = h * rows_per_head;  // original Q rows of head h
            // post the byte count before any lane's copy can complete_tx
            if (lane == 0) mbar_arrive_expect_tx(&sm.q_full, hasB ? 2 * TILE_BYTES : TILE_BYTES);
            __syncwarp();
            for (int t = 0; t < (hasB ? 2 : 1); ++t) {
                int a0, a1, a2, a3;
                rows4((tA + t) * BM + 4 * (int)lane, a0, a1, a2, a3);
                uint8_t* dst = sm.q[t] + lane * 512;
                tma_gather4(dst, &tm_q, &sm.q_full, 0, q_base_row + a0, q_base_row + a1,
                            q_base_row + a2, q_base_row + a3);
                tma_gather4(dst + HALF_BYTES, &tm_q, &sm.q_full, 64, q_base_row + a0,
                            q_base_row + a1, q_base_row + a2, q_base_row + a3);
            }
            // K/V: tiled loads of the compressed per-head buffers (kc/vc from the
            // gather kernel) -- 4 TMA requests per KV step instead of 128 gathers.
            // k_keep == L (tau = 0): the selection is the identity, so the tiles
            // come straight from the KV head's rows (no compressed copy, and the
            // query heads of a KV group share them in L2 as the dense kernel does)
            // (Two copies of the loop, each on a fixed descriptor: selecting the
            // descriptor address at run time measured 3 % slower on the whole
            // attention.)
            auto kv_loop = [&](const CUtensorMap& mk, const CUtensorMap& mv, const CUtensorMap& mv3,
                               int head) {
                const int row0 = head * rows_per_head;
                for (int j = 0; j < nkv; ++j) {
                    const int st = j % NS;
                    const int r = j * BN;
                    if (j >= NS) mbar_wait(&sm.k_empty[st], ((j / NS) - 1) & 1);
                    tma_load_2d(sm.k[st], &mk, &sm.k_full[st], 0, row0 + r);
                    tma_load_2d(sm.k[st] + HALF_BYTES, &mk, &sm.k_full[st], 64, row0 + r);
                    mbar_arrive_expect_tx(&sm.k_full[st], TILE_BYTES);
                    if (j >= NS) mbar_wait(&sm.v_empty[st], ((j / NS) - 1) & 1);
                    if (r + BN <= rows_per_head) {
                        tma_load_2d(sm.v[st], &mv, &sm.v_full[st], 0, row0 + r);
                        tma_load_2d(sm.v[st] + HALF_BYTES, &mv, &sm.v_full[st], 64, row0 + r);
                    } else {  // past the head's rows: zeros (3-D map)
                        tma_load_3d(sm.v[st], &mv3, &sm.v_full[st], 0, r, head);
                        tma_load_3d(sm.v[st] + HALF_BYTES, &mv3, &sm.v_full[st], 64, r, head);
                    }
                    mbar_arrive_expect_tx(&sm.v_full[st], TILE_BYTES);
                }
            };
            if (lane == 0) {
                if (n == rows_per_head)
                    kv_loop(tm_kd, tm_vd, tm_vd3, h / dense_group);
                else
                    kv_loop(tm_k, tm_v, tm_v3, kvh);
            }
        }
    } else if (warp == 9) {
        // ------------------------------------------------------ MMA issuer
        {  // the whole warp runs the loop (warp-uniform state); the elected lane issues
            const uint32_t L1 = elect_one() ? 1u : 0u;
            const uint32_t idesc_s = idesc_bf16_f32(BM, BN, 0, 0);
            const uint32_t idesc_o = idesc_bf16_f32(BM, HD, 0, 1);
            const uint32_t qa = smem_u32(sm.q[0]), qb = smem_u32(sm.q[1]);
            // (Keep this warp's register footprint small: when other roles of the
            // kernel grow, ptxas can move the TMEM addresses out of uniform
            // registers and every TS-MMA then pays an R2UR.BROADCAST -- the SASS
            // of both instantiations is checked by tests/test_sass.py.)
            const uint32_t tS[2] = {tmem, tmem + 128};
            const uint32_t tO[2] = {tmem + 256, tmem + 384};
            auto doA = [&](int j) { return j <= tA; };
            auto doB = [&](int j) { return hasB && j <= tB; };
            mbar_wait(&sm.q_full, 0);
            // prologue: S(0) for both tiles
            mbar_wait(&sm.k_full[0], 0);
            tc_fence_after();
            issue_s(tS[0], qa, smem_u32(sm.k[0]), idesc_s, L1);
            mma_commit_p(&sm.s_full[0], L1);
            if (hasB) {
                issue_s(tS[1], qb, smem_u32(sm.k[0]), idesc_s, L1);
                mma_commit_p(&sm.s_full[1], L1);
            }
            mma_commit_p(&sm.k_empty[0], L1);
            for (int j = 0; j < nkv; ++j) {
                const int st = j % NS;
                const int j1 = j + 1, st1 = j1 % NS;
                mbar_wait(&sm.v_full[st], (j / NS) & 1);
                const uint32_t v_base = smem_u32(sm.v[st]);
                const bool k1_needed = (j1 < nkv) && (doA(j1) || doB(j1));
                if (doA(j)) {
#pragma unroll
                    for (int qq = 0; qq < 4; ++qq) {
                        mbar_wait(&sm.p_full[0][qq], j & 1);
                        tc_fence_after();
                        issue_pv_quarter(tO[0], tS[0], v_base, idesc_o, j > 0, qq, L1);
                    }
                    mma_commit_p(&sm.o_done[0], L1);
                    if (doA(j1)) {
                        mbar_wait(&sm.k_full[st1], (j1 / NS) & 1);
                        tc_fence_after();
                        issue_s(tS[0], qa, smem_u32(sm.k[st1]), idesc_s, L1);
                        mma_commit_p(&sm.s_full[0], L1);
                    }
                }
                if (doB(j)) {
#pragma unroll
                    for (int qq = 0; qq < 4; ++qq) {
                        mbar_wait(&sm.p_full[1][qq], j & 1);
                        tc_fence_after();
                        issue_pv_quarter(tO[1], tS[1], v_base, idesc_o, j > 0, qq, L1);
                    }
                    mma_commit_p(&sm.o_done[1], L1);
                    if (doB(j1)) {
                        mbar_wait(&sm.k_full[st1], (j1 / NS) & 1);
                        tc_fence_after();
                        issue_s(tS[1], qb, smem_u32(sm.k[st1]), idesc_s, L1);
                        mma_commit_p(&sm.s_full[1], L1);
                    }
                }
                if (k1_needed) mma_commit_p(&sm.k_empty[st1], L1);
                mma_commit_p(&sm.v_empty[st], L1);
            }
        }
        // teardown: wait for the softmax warps' last TMEM reads, then free TMEM
        named_bar_sync(1, 288);
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}
// ------------------------------------------------------------------ host
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

}  // namespace

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() { return encode_fn(); }

// 2-D map over a [rows x 128] bf16 matrix, 64-column x box_rows boxes, 128-B swizzle.
int make_bf16_map_2d(CUtensorMap* m, const void* base, uint64_t rows, uint32_t box_rows) {
    auto fn = encode_fn();
    if (!fn) return invalid("tsa: cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {HD, rows};
    cuuint64_t strides[1] = {HD * 2};
    cuuint32_t box[2] = {64, box_rows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                    box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        return invalid("tsa: tensor map encode failed (" + std::to_string((int)r) + ")");
    return 0;
}

// 2-D map over an f32 matrix [rows x inner] (row pitch row_stride_bytes, a
// multiple of 16), box_inner x box_rows boxes, no swizzle (score_exact.cu).
int make_f32_map_2d(CUtensorMap* m, const void* base, uint64_t inner, uint64_t rows,
                    uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_rows) {
    auto fn = encode_fn();
    if (!fn) return invalid("tsa: cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {inner, rows};
    cuuint64_t strides[1] = {row_stride_bytes};
    cuuint32_t box[2] = {box_inner, box_rows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides,
                    box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        return invalid("tsa: f32 tensor map encode failed (" + std::to_string((int)r) + ")");
    return 0;
}

// 2-D map over [rows x 128] bf16 rows, whole-row (256 B) x box_rows boxes, no
// swizzle: rows land in shared memory back to back (gather_scatter.cu's TMA
// gather: tile::gather4 loads with box_rows = 1, bulk tensor stores of 64 rows).
int make_bf16_rows_map(CUtensorMap* m, const void* base, uint64_t rows, uint32_t box_rows) {
    auto fn = encode_fn();
    if (!fn) return invalid("tsa: cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {HD, rows};
    cuuint64_t strides[1] = {HD * 2};
    cuuint32_t box[2] = {HD, box_rows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                    box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        return invalid("tsa: row tensor map encode failed (" + std::to_string((int)r) + ")");
    return 0;
}

// 3-D [heads x rows x 128] bf16, whole-row x box_rows x 1 boxes, no swizzle: a
// store box never crosses into the next head (rows >= `rows` are clipped).
int make_bf16_rows_map_3d(CUtensorMap* m, const void* base, uint64_t rows, uint64_t heads,
                          uint32_t box_rows) {
    auto fn = encode_fn();
    if (!fn) return invalid("tsa: cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[3] = {HD, rows, heads};
    cuuint64_t strides[2] = {HD * 2, rows * HD * 2};
    cuuint32_t box[3] = {HD, box_rows, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides,
                    box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        return invalid("tsa: 3-D row tensor map encode failed (" + std::to_string((int)r) + ")");
    return 0;
}

// 3-D map over [heads x rows x 128] bf16 with the same 64 x 128 SW128 boxes,
// used by the indexed kernel for a head's last, partial V tile: past the
// head's last row it reads zeros (out of bounds), never the next head's rows
// -- which may not have arrived yet (the host-tensor pipeline copies V per
// head group) or hold anything at all; those keys are masked, but P = 0 times
// a NaN still poisons O.  (Only the partial tile: 3-D loads for every tile
// measured ~1 % slower.)
int make_bf16_map_3d(CUtensorMap* m, const void* base, uint64_t rows, uint64_t heads) {
    auto fn = encode_fn();
    if (!fn) return invalid("tsa: cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[3] = {HD, rows, heads};
    cuuint64_t strides[2] = {HD * 2, rows * HD * 2};
    cuuint32_t box[3] = {64, 128, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides,
                    box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        return invalid("tsa: tensor map encode failed (" + std::to_string((int)r) + ")");
    return 0;
}

bool attend_sm100_supported(const tsa_desc& d) { return d.dtype == TSA_BF16 && d.d_head == HD; }

namespace {

// Which exponential pairs of each 32-key chunk run on the FMA pipe
// (TSA_EXP_POLY = 0 / 25 / 37 / 50 percent).  Default 25: with the current
// kernel a quarter of the off-diagonal exponentials on the FMA pipe measured
// -1.8 % at 128K (dense -1.3 %; profiles/r1/ab_exp_poly.log); 12.5 / 18.75 /
// 37.5 / 50 % all measured slower than 25 %;
// the diagonal tile always uses MUFU.  (An earlier revision measured 25 %
// slower: profiles/r1/poly_sweep.log.)
uint32_t poly_mask() {
    static const uint32_t m = [] {
        const char* e = std::getenv("TSA_EXP_POLY");
        const int pct = e ? std::atoi(e) : 25;
        return pct <= 0 ? 0x0000u : pct <= 25 ? 0x1111u : pct <= 37 ? 0x2929u : 0x5555u;
    }();
    return m;
}

template <bool kIndexed, uint32_t kPolyMask>
void run_kernel(dim3 grid, cudaStream_t st, const CUtensorMap& mq, const CUtensorMap& mk,
                const CUtensorMap& mv, const CUtensorMap& mkd, const CUtensorMap& mvd,
                const CUtensorMap& mv3, const CUtensorMap& mvd3, int dense_group, const int32_t* n_dev, int32_t n_const, int32_t kv_group,
                int32_t rows_per_head, int32_t kv_rows_per_head, int head_begin, float scale_log2,
                const OutReplicas& o, const int32_t* idx) {
    const int smem = (int)sizeof(AttnSmem) + 1024;
    ensure_smem_attr(reinterpret_cast<const void*>(attend_sm100_kernel<kIndexed, kPolyMask>), smem);
    attend_sm100_kernel<kIndexed, kPolyMask><<<grid, kThreads, smem, st>>>(
        mq, mk, mv, mkd, mvd, mv3, mvd3, dense_group, n_dev, n_const, kv_group, rows_per_head,
        kv_rows_per_head, head_begin,
        scale_log2, o, idx);
}

template <bool kIndexed>
int launch_impl(const tsa_desc& d, const void* q, const void* k, const void* v,
                const void* k_dense, const void* v_dense,
                const int32_t* idx, const int32_t* n_dev, int32_t n_const, int32_t kv_group,
                int32_t rows_per_head, int32_t kv_rows_per_head, const OutReplicas& o,
                cudaStream_t st) {
    if (!attend_sm100_supported(d)) return invalid("attend_sm100: needs bf16, d_head 128");
    const int nh = d.head_end - d.head_begin;
    const int n_q_heads = d.n_heads;
    const int n_kv_heads_buf = (n_q_heads + kv_group - 1) / kv_group;
    CUtensorMap mq, mk, mv;
    int rc;
    // the gather4 Q map uses one-row boxes
    if ((rc = make_bf16_map_2d(&mq, q, (uint64_t)n_q_heads * rows_per_head, kIndexed ? 1 : 128)))
        return rc;
    if ((rc = make_bf16_map_2d(&mk, k, (uint64_t)n_kv_heads_buf * kv_rows_per_head, 128))) return rc;
    if ((rc = make_bf16_map_2d(&mv, v, (uint64_t)n_kv_heads_buf * kv_rows_per_head, 128))) return rc;
    CUtensorMap mv3;  // V's last partial tile per head (zeros past the head's rows)
    if ((rc = make_bf16_map_3d(&mv3, v, (uint64_t)kv_rows_per_head, (uint64_t)n_kv_heads_buf)))
        return rc;
    // the KV heads in place (indexed path, k_keep == L); the compressed maps otherwise
    CUtensorMap mkd = mk, mvd = mv, mvd3 = mv3;
    const int dense_group = d.n_heads / d.n_kv_heads;
    if (kIndexed && k_dense && v_dense) {
        if ((rc = make_bf16_map_2d(&mkd, k_dense, (uint64_t)d.n_kv_heads * rows_per_head, 128)))
            return rc;
        if ((rc = make_bf16_map_2d(&mvd, v_dense, (uint64_t)d.n_kv_heads * rows_per_head, 128)))
            return rc;
        if ((rc = make_bf16_map_3d(&mvd3, v_dense, (uint64_t)rows_per_head, (uint64_t)d.n_kv_heads)))
            return rc;
    }
    const int max_tiles = (rows_per_head + BM - 1) / BM;
    dim3 grid((max_tiles + 1) / 2, nh);
    const float scale_log2 = (1.0f / sqrtf((float)HD)) * 1.4426950408889634f;
    switch (poly_mask()) {
        case 0x0000u:
            run_kernel<kIndexed, 0x0000u>(grid, st, mq, mk, mv, mkd, mvd, mv3, mvd3, dense_group, n_dev, n_const, kv_group,
                                          rows_per_head, kv_rows_per_head, d.head_begin,
                                          scale_log2, o, idx);
            break;
        case 0x1111u:
            run_kernel<kIndexed, 0x1111u>(grid, st, mq, mk, mv, mkd, mvd, mv3, mvd3, dense_group, n_dev, n_const, kv_group,
                                          rows_per_head, kv_rows_per_head, d.head_begin,
                                          scale_log2, o, idx);
            break;
        case 0x5555u:
            run_kernel<kIndexed, 0x5555u>(grid, st, mq, mk, mv, mkd, mvd, mv3, mvd3, dense_group, n_dev, n_const, kv_group,
                                          rows_per_head, kv_rows_per_head, d.head_begin,
                                          scale_log2, o, idx);
            break;
        default:
            run_kernel<kIndexed, 0x2929u>(grid, st, mq, mk, mv, mkd, mvd, mv3, mvd3, dense_group, n_dev, n_const, kv_group,
                                          rows_per_head, kv_rows_per_head, d.head_begin,
                                          scale_log2, o, idx);
    }
    TSA_LAUNCH_CHECK(kIndexed ? "attend_sm100_indexed" : "attend_sm100");
    return 0;
}

}  // namespace

int launch_attend_sm100(const tsa_desc& d, const void* q, const void* k, const void* v,
                        const int32_t* n_dev, int32_t n_const, int32_t kv_group,
                        int32_t rows_per_head, int32_t kv_rows_per_head, void* o,
                        cudaStream_t st) {
    return launch_impl<false>(d, q, k, v, nullptr, nullptr, nullptr, n_dev, n_const, kv_group,
                              rows_per_head, kv_rows_per_head, single_replica(o), st);
}

// Dense causal attention with the output rows stored to every replica (the
// head-sharded dense layer's all-gather fused into the epilogue).
int launch_attend_sm100_rep(const tsa_desc& d, const void* q, const void* k, const void* v,
                            const OutReplicas& o, cudaStream_t st) {
    const int L = d.seq_len;
    return launch_impl<false>(d, q, k, v, nullptr, nullptr, nullptr, nullptr, L,
                              d.n_heads / d.n_kv_heads, L, L, o, st);
}

// Fused gather -> causal attention -> scatter of the selected rows (the
// unselected rows are zeroed separately by launch_zero_unselected).
int launch_attend_indexed(const tsa_desc& d, const void* q, const void* k, const void* v,
                          const void* kc, const void* vc, const int32_t* idx,
                          const int32_t* k_keep, void* out, cudaStream_t st) {
    const int L = d.seq_len;
    return launch_impl<true>(d, q, kc, vc, k, v, idx, k_keep, L, 1, L, L, single_replica(out), st);
}

// The same with the output rows stored to every replica (tsa_attend_indexed_replicas).
int launch_attend_indexed_rep(const tsa_desc& d, const void* q, const void* k, const void* v,
                              const void* kc, const void* vc, const int32_t* idx,
                              const int32_t* k_keep, const OutReplicas& out, cudaStream_t st) {
    const int L = d.seq_len;
    return launch_impl<true>(d, q, kc, vc, k, v, idx, k_keep, L, 1, L, L, out, st);
}

}  // namespace tsa
