// K5 for f32 (cfg1): causal attention on the tensor cores at f32 accuracy.
//
// dense_causal_attention (attention.cpp:25-40) in f32 with the reference's
// 1e-5 gate (bench.cpp:27): a single TF32 product keeps ~11 mantissa bits, so
// every product is split "3xTF32": x = hi + lo with hi = x with its 13 low
// mantissa bits cleared (exact in TF32) and lo = x - hi (exact in f32, |lo| <
// 2^-10 |x|), and a.b ~= hi.hi + hi.lo + lo.hi (the dropped lo.lo term is
// ~2^-20 relative) -- three kind::tf32 MMAs accumulating in f32 in TMEM.
//
// One CTA per 128-row query tile (heaviest first), 10 warps:
//   warp 0      TMA producer: the Q tile once (4 chunks of 32 columns), then
//               per KV tile 4 K chunks [128 keys x 32 dims] and 4 V chunks
//               [32 keys x 128 dims] through a 3-stage ring (raw f32, 128-B
//               swizzle; 3-D maps, so rows past a head read zeros), in the
//               MMA's order K(0), K(1) V(0), K(2) V(1), ...
//   warp 1      MMA issuer: S(j) = Q K_j^T as 48 SS-MMAs M128 N128 K8 (3 per
//               k-step) into one of two S buffers, O += P(j) V_j as 48 TS-MMAs
//               (P from TMEM, V MN-major); order S(0) S(1) | PV(0) S(2) |
//               PV(1) S(3) ..., so the tensor core computes PV(j) and S(j+2)
//               while the softmax works on tile j+1
//   warps 2-5   split: raw chunk -> hi in place + lo beside it (elementwise,
//               so the swizzled layout is kept), then fence.proxy.async
//   warps 6-9   softmax, thread = row = TMEM lane: row max (pass 1 over S in
//               TMEM), p = exp(s - m) with causal masking, O rescaled when
//               the max grows, row sum, P_hi over S and P_lo beside it
//               (tcgen05.st); epilogue O / l -> global.
// TMEM: S / P_hi in two buffers [0,128) [128,256), P_lo [256,384), O
// [384,512).  S(j+2) reuses the buffer PV(j) reads P_hi(j) from: the MMAs
// execute in issue order.  The softmax of tile j+1 finds its row max while
// PV(j) runs and waits for PV(j) only before it rescales O and writes P_lo.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>

#include "common.cuh"
#include "sm100.cuh"

namespace tsa {

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder();

namespace {

using namespace tsa_dev;

constexpr int TBM = 128;                   // query rows per tile / keys per KV tile
constexpr int TD = 128;                    // head dim
constexpr int CHUNK_BYTES = 128 * 32 * 4;  // [128 x 32] f32 = 16 KiB
constexpr int NSTG = 3;
constexpr int kTf32Threads = 320;
// exp(x) = 2^(x log2 e) on MUFU.EX2 (rel. error ~2^-22; the argument's rounding
// adds |x| 2^-24 relative -- both far inside the 1e-5 gate)
constexpr float kLog2e = 1.4426950408889634f;

struct __align__(1024) Tf32Smem {
    uint8_t q_hi[4][CHUNK_BYTES];  // Q chunk c: dims [32c, 32c + 32)
    uint8_t q_lo[4][CHUNK_BYTES];
    uint8_t hi[NSTG][CHUNK_BYTES];  // raw, then hi in place
    uint8_t lo[NSTG][CHUNK_BYTES];
    uint64_t q_full, q_ready;
    uint64_t raw_full[NSTG], conv_full[NSTG], empty[NSTG];
    uint64_t s_full[2], p_full, pv_done;
    uint32_t tmem_base;
};

// kind::tf32: D f32, A / B TF32, M 128, N 128.
__host__ __device__ constexpr uint32_t idesc_tf32(uint32_t b_mn_major, uint32_t m = 128) {
    return (1u << 4) | (2u << 7) | (2u << 10) | (b_mn_major << 16) | ((128u >> 3) << 17) |
           ((m >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32_ss_p(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                              uint32_t idesc, uint32_t accumulate, uint32_t issue) {
    asm volatile(
        "{\n"
        ".reg .pred p, q;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "setp.ne.b32 q, %5, 0;\n"
        "@q tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate), "r"(issue)
        : "memory");
}
__device__ __forceinline__ void mma_tf32_ts_p(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                              uint32_t idesc, uint32_t accumulate, uint32_t issue) {
    asm volatile(
        "{\n"
        ".reg .pred p, q;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "setp.ne.b32 q, %5, 0;\n"
        "@q tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n"
        "}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate), "r"(issue)
        : "memory");
}

// K-major SW128 (LBO 16 B, SBO 1 KiB): one 128-B row = 32 f32 of K.
__device__ __forceinline__ uint64_t kdesc(uint32_t saddr) {
    return (static_cast<uint64_t>(0x40004040u) << 32) | (((saddr >> 4) & 0x3FFFu) | (1u << 16));
}
// MN-major TF32: 128-B rows = 32 f32 of N, one row per K, swizzled in 32-B
// atoms (layout 1, SWIZZLE_128B_BASE32B; TMA SWIZZLE_128B_ATOM_32B), 4-row K
// groups 512 B apart (SBO), N atoms 4 KiB apart (LBO).  The plain 128-B
// swizzle reads as zeros for MN-major TF32 (tools/probes/tf32_probe.cu).
__device__ __forceinline__ uint64_t ndesc(uint32_t saddr) {
    constexpr uint32_t hi = (1u << 29) | (1u << 14) | (512u >> 4);
    return (static_cast<uint64_t>(hi) << 32) | (((saddr >> 4) & 0x3FFFu) | ((4096u >> 4) << 16));
}

__device__ __forceinline__ float tf32_hi(float x) {
    return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}

// 16 KiB raw chunk -> hi in place, lo into `lo`; 128 threads, 8 x 16 B each
// (shared-window addresses: LDS / STS, not generic loads).
template <int BYTES = CHUNK_BYTES>
__device__ __forceinline__ void split_chunk(uint8_t* hi, uint8_t* lo, uint32_t t) {
    const uint32_t h0 = smem_u32(hi), l0 = smem_u32(lo);
    float4 x[BYTES / 16 / 128];
#pragma unroll
    for (int i = 0; i < BYTES / 16 / 128; ++i)
        asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(x[i].x), "=f"(x[i].y), "=f"(x[i].z), "=f"(x[i].w)
                     : "r"(h0 + (i * 128 + t) * 16));
#pragma unroll
    for (int i = 0; i < BYTES / 16 / 128; ++i) {
        const uint32_t off = (i * 128 + t) * 16;
        const float4 h = make_float4(tf32_hi(x[i].x), tf32_hi(x[i].y), tf32_hi(x[i].z), tf32_hi(x[i].w));
        asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(h0 + off), "f"(h.x), "f"(h.y),
                     "f"(h.z), "f"(h.w)
                     : "memory");
        asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(l0 + off), "f"(x[i].x - h.x),
                     "f"(x[i].y - h.y), "f"(x[i].z - h.z), "f"(x[i].w - h.w)
                     : "memory");
    }
}

__global__ void __launch_bounds__(kTf32Threads, 1)
attend_tf32_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                   const __grid_constant__ CUtensorMap tm_v, const int32_t* __restrict__ n_dev,
                   int n_const, int kv_group, int rows_per_head, int head_begin, float scale,
                   float* __restrict__ o, const int32_t* __restrict__ o_rows) {
    extern __shared__ uint8_t smem_raw[];
    Tf32Smem& sm = *reinterpret_cast<Tf32Smem*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    // grid (heads, tile slots): the launch order walks every head's heaviest
    // tile before any head's next one (longest-first over the whole layer)
    const int h = head_begin + blockIdx.x;
    const int n = n_dev ? *n_dev : n_const;
    const int n_tiles = (n + TBM - 1) / TBM;
    if ((int)blockIdx.y >= n_tiles) return;
    const int t = n_tiles - 1 - (int)blockIdx.y;  // heaviest tiles first
    const int nkv = t + 1;
    const int kvh = h / kv_group;
    const uint32_t warp = warp_id_uniform();
    const uint32_t lane = lane_id();

    if (threadIdx.x == 0) {
        mbar_init(&sm.q_full, 1);
        mbar_init(&sm.q_ready, 128);
        for (int s = 0; s < NSTG; ++s) {
            mbar_init(&sm.raw_full[s], 1);
            mbar_init(&sm.conv_full[s], 128);
            mbar_init(&sm.empty[s], 1);
        }
        mbar_init(&sm.s_full[0], 1);
        mbar_init(&sm.s_full[1], 1);
        mbar_init(&sm.p_full, 128);
        mbar_init(&sm.pv_done, 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(&sm.tmem_base, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sm.tmem_base;
    const uint32_t t_lo = tmem + 256, t_o = tmem + 384;  // S buffers at tmem + 128 b
    const int n_items = nkv * 8;  // per KV tile: 4 K chunks and 4 V chunks

    if (warp == 0) {
        // ---------------------------------------------------------------- TMA
        if (lane == 0) {
            mbar_arrive_expect_tx(&sm.q_full, 4 * CHUNK_BYTES);
            for (int c = 0; c < 4; ++c) tma_load_3d(sm.q_hi[c], &tm_q, &sm.q_full, 32 * c, t * TBM, h);
            int it = 0;
            auto load = [&](int j, bool is_v) {
                for (int c = 0; c < 4; ++c, ++it) {
                    const int s = it % NSTG;
                    if (it >= NSTG) mbar_wait(&sm.empty[s], ((it / NSTG) - 1) & 1);
                    mbar_arrive_expect_tx(&sm.raw_full[s], CHUNK_BYTES);
                    if (!is_v) {
                        tma_load_3d(sm.hi[s], &tm_k, &sm.raw_full[s], 32 * c, j * TBM, kvh);
                    } else {  // V keys [32 c, +32) of tile j: four N atoms of 32 dims
                        for (int a = 0; a < 4; ++a)
                            tma_load_3d(sm.hi[s] + a * 4096, &tm_v, &sm.raw_full[s], 32 * a,
                                        j * TBM + 32 * c, kvh);
                    }
                }
            };
            load(0, false);
            for (int j = 0; j < nkv; ++j) {
                if (j + 1 < nkv) load(j + 1, false);
                load(j, true);
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ---------------------------------------------------------------- MMA
        const uint32_t issue = elect_one() ? 1u : 0u;
        constexpr uint32_t id_s = idesc_tf32(0), id_pv = idesc_tf32(1);
        mbar_wait(&sm.q_ready, 0);
        tc_fence_after();
        int it = 0;
        auto issue_s = [&](int j) {
            const uint32_t t_s = tmem + 128 * (j & 1);
            for (int c = 0; c < 4; ++c, ++it) {
                const int s = it % NSTG;
                mbar_wait(&sm.conv_full[s], (it / NSTG) & 1);
                tc_fence_after();
                const uint32_t qh = smem_u32(sm.q_hi[c]), ql = smem_u32(sm.q_lo[c]);
                const uint32_t kh = smem_u32(sm.hi[s]), kl = smem_u32(sm.lo[s]);
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    const uint32_t off = kk * 32;
                    mma_tf32_ss_p(t_s, kdesc(qh + off), kdesc(kh + off), id_s, (c | kk) ? 1u : 0u, issue);
                    mma_tf32_ss_p(t_s, kdesc(qh + off), kdesc(kl + off), id_s, 1u, issue);
                    mma_tf32_ss_p(t_s, kdesc(ql + off), kdesc(kh + off), id_s, 1u, issue);
                }
                mma_commit_p(&sm.empty[s], issue);
            }
            mma_commit_p(&sm.s_full[j & 1], issue);
        };
        issue_s(0);
        for (int j = 0; j < nkv; ++j) {
            if (j + 1 < nkv) issue_s(j + 1);
            mbar_wait(&sm.p_full, j & 1);
            tc_fence_after();
            const uint32_t t_p = tmem + 128 * (j & 1);
            for (int c = 0; c < 4; ++c, ++it) {
                const int s = it % NSTG;
                mbar_wait(&sm.conv_full[s], (it / NSTG) & 1);
                tc_fence_after();
                const uint32_t vh = smem_u32(sm.hi[s]), vl = smem_u32(sm.lo[s]);
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    const uint32_t col = c * 32 + kk * 8, off = kk * 1024;
                    mma_tf32_ts_p(t_o, t_p + col, ndesc(vh + off), id_pv, (j | c | kk) ? 1u : 0u, issue);
                    mma_tf32_ts_p(t_o, t_p + col, ndesc(vl + off), id_pv, 1u, issue);
                    mma_tf32_ts_p(t_o, t_lo + col, ndesc(vh + off), id_pv, 1u, issue);
                }
                mma_commit_p(&sm.empty[s], issue);
            }
            mma_commit_p(&sm.pv_done, issue);
        }
    } else if (warp < 6) {
        // ---------------------------------------------------------------- split
        const uint32_t tid = threadIdx.x - 64;
        mbar_wait(&sm.q_full, 0);
        for (int c = 0; c < 4; ++c) split_chunk(sm.q_hi[c], sm.q_lo[c], tid);
        fence_proxy_async_smem();
        mbar_arrive(&sm.q_ready);
        for (int it = 0; it < n_items; ++it) {
            const int s = it % NSTG;
            mbar_wait(&sm.raw_full[s], (it / NSTG) & 1);
            split_chunk(sm.hi[s], sm.lo[s], tid);
            fence_proxy_async_smem();
            mbar_arrive(&sm.conv_full[s]);
        }
    } else {
        // ---------------------------------------------------------------- softmax
        const uint32_t quarter = warp & 3;
        const int row = t * TBM + (int)(quarter * 32 + lane);  // row within the head
        const uint32_t lane_off = (quarter * 32) << 16;
        float m = -INFINITY, l = 0.0f;
        for (int j = 0; j < nkv; ++j) {
            const uint32_t t_s = tmem + 128 * (j & 1);
            mbar_wait(&sm.s_full[j & 1], (j >> 1) & 1);
            tc_fence_after();
            const bool diag = j == t;
            // pass 1: row max of the scaled, masked logits (the four 32-column
            // loads in flight together, one wait)
            float mx = -INFINITY;
            {
                uint32_t sr[128];
                tmem_ld32_at<0>(t_s + lane_off, sr);
                tmem_ld32_at<32>(t_s + lane_off + 32, sr);
                tmem_ld32_at<64>(t_s + lane_off + 64, sr);
                tmem_ld32_at<96>(t_s + lane_off + 96, sr);
                tmem_wait_ld();
#pragma unroll
                for (int e = 0; e < 128; ++e) {
                    const int key = j * TBM + e;
                    const float x = __fmul_rn(__uint_as_float(sr[e]), scale);
                    if (!diag || key <= row) mx = fmaxf(mx, x);
                }
            }
            if (j > 0) {  // PV(j-1) done: O is final through tile j-1, P_lo is free
                mbar_wait(&sm.pv_done, (j - 1) & 1);
                tc_fence_after();
            }
            const float m_new = fmaxf(m, mx);
            const float corr = (m == -INFINITY) ? 0.0f : ex2_approx(__fmul_rn(m - m_new, kLog2e));
            // O rescaled when the max grew
            if (j > 0 && __any_sync(0xffffffffu, corr != 1.0f)) {
#pragma unroll 1
                for (int c = 0; c < 4; ++c) {
                    uint32_t r[32];
                    tmem_ld32(t_o + lane_off + c * 32, r);
                    tmem_wait_ld();
#pragma unroll
                    for (int e = 0; e < 32; ++e) r[e] = __float_as_uint(__uint_as_float(r[e]) * corr);
                    tmem_st32(t_o + lane_off + c * 32, r);
                }
            }
            l *= corr;
            m = m_new;
            // pass 2: p, the row sum, P_hi over S and P_lo beside it (64 columns
            // loaded per wait)
#pragma unroll 1
            for (int hc = 0; hc < 2; ++hc) {
                uint32_t sr[64];
                tmem_ld32_at<0>(t_s + lane_off + hc * 64, sr);
                tmem_ld32_at<32>(t_s + lane_off + hc * 64 + 32, sr);
                tmem_wait_ld();
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    uint32_t rh[32], rl[32];
#pragma unroll
                    for (int e = 0; e < 32; ++e) {
                        const int key = j * TBM + hc * 64 + c * 32 + e;
                        const float x = __fmul_rn(__uint_as_float(sr[c * 32 + e]), scale);
                        const float p = (!diag || key <= row) ? ex2_approx(__fmul_rn(x - m, kLog2e)) : 0.0f;
                        l += p;
                        const float ph = tf32_hi(p);
                        rh[e] = __float_as_uint(ph);
                        rl[e] = __float_as_uint(p - ph);
                    }
                    tmem_st32(t_s + lane_off + hc * 64 + c * 32, rh);
                    tmem_st32(t_lo + lane_off + hc * 64 + c * 32, rl);
                }
            }
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(&sm.p_full);
        }
        mbar_wait(&sm.pv_done, (nkv - 1) & 1);
        tc_fence_after();
        const float inv_l = 1.0f / l;
        // o_rows: the decompress fused -- kept row `row` lands at its original position
        const int orow = (o_rows && row < n) ? __ldg(o_rows + (size_t)h * rows_per_head + row) : row;
        float* dst = o + ((size_t)h * rows_per_head + orow) * TD;
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
            uint32_t r[32];
            tmem_ld32(t_o + lane_off + c * 32, r);
            tmem_wait_ld();
            if (row < n) {
#pragma unroll
                for (int e = 0; e < 32; e += 4)
                    *reinterpret_cast<float4*>(dst + c * 32 + e) =
                        make_float4(__uint_as_float(r[e]) * inv_l, __uint_as_float(r[e + 1]) * inv_l,
                                    __uint_as_float(r[e + 2]) * inv_l, __uint_as_float(r[e + 3]) * inv_l);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, 512);
}

// ---------------------------------------------------------------- CTA pairs
// The same attention on 2-CTA clusters (cta_group::2): the pair's two CTAs
// hold query tiles 2p and 2p+1 of a head (128 rows each, M = 256 per MMA) and
// share every K / V chunk -- each CTA stages and splits only its half (64 keys
// of a K chunk, 64 dims of a V chunk) and the tensor cores exchange the B
// halves.  Per SM this halves the B-operand shared-memory reads, the split
// work and the TMA bytes: the single-CTA kernel's S MMA reads A and B at
// 128 B/clk, the whole shared-memory bandwidth, so it cannot keep the tensor
// pipe busy (ncu: 45 %).  The pair walks KV tiles 0..2p+1; tile 2p+1 is fully
// masked for the lower tile (its MMA work is the price of sharing).
// The leader (cluster rank 0) issues the MMAs; the split and softmax threads
// of both CTAs arrive on the leader's barriers; the MMA commits multicast to
// both CTAs.
constexpr int HALF_BYTES = CHUNK_BYTES / 2;  // [64 x 32] f32 = 8 KiB
constexpr int NSTG2 = 6;

struct __align__(1024) Tf32PairSmem {
    uint8_t q_hi[4][CHUNK_BYTES];
    uint8_t q_lo[4][CHUNK_BYTES];
    uint8_t hi[NSTG2][HALF_BYTES];
    uint8_t lo[NSTG2][HALF_BYTES];
    uint64_t q_full, q_ready;
    uint64_t raw_full[NSTG2], conv_full[NSTG2], empty[NSTG2];
    uint64_t s_full[2], p_full, pv_done;
    uint32_t tmem_base;
};

__device__ __forceinline__ void mma_tf32_ss_pair_p(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                                   uint32_t idesc, uint32_t accumulate,
                                                   uint32_t issue) {
    asm volatile(
        "{\n"
        ".reg .pred p, q;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "setp.ne.b32 q, %5, 0;\n"
        "@q tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate), "r"(issue)
        : "memory");
}
__device__ __forceinline__ void mma_tf32_ts_pair_p(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                                   uint32_t idesc, uint32_t accumulate,
                                                   uint32_t issue) {
    asm volatile(
        "{\n"
        ".reg .pred p, q;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "setp.ne.b32 q, %5, 0;\n"
        "@q tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n"
        "}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate), "r"(issue)
        : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kTf32Threads, 1)
attend_tf32_pair_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                        const __grid_constant__ CUtensorMap tm_v, const int32_t* __restrict__ n_dev,
                        int n_const, int kv_group, int rows_per_head, int head_begin, float scale,
                        float* __restrict__ o, const int32_t* __restrict__ o_rows) {
    extern __shared__ uint8_t smem_raw[];
    Tf32PairSmem& sm = *reinterpret_cast<Tf32PairSmem*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    // grid (2 x heads, pair slots), clusters along x: longest-first over the layer
    const int h = head_begin + ((int)blockIdx.x >> 1);
    const int n = n_dev ? *n_dev : n_const;
    const int n_tiles = (n + TBM - 1) / TBM;
    const int n_pairs = (n_tiles + 1) / 2;
    const int cid = (int)blockIdx.y;
    if (cid >= n_pairs) return;  // uniform over the pair
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;
    const int p = n_pairs - 1 - cid;  // heaviest pairs first
    const int t = 2 * p + (int)rank;  // this CTA's query tile
    const int nkv = min(2 * p + 2, n_tiles);
    const int kvh = h / kv_group;
    const uint32_t warp = warp_id_uniform();
    const uint32_t lane = lane_id();

    if (threadIdx.x == 0) {
        mbar_init(&sm.q_full, 1);
        mbar_init(&sm.q_ready, 256);
        for (int s = 0; s < NSTG2; ++s) {
            mbar_init(&sm.raw_full[s], 1);
            mbar_init(&sm.conv_full[s], 256);
            mbar_init(&sm.empty[s], 1);
        }
        mbar_init(&sm.s_full[0], 1);
        mbar_init(&sm.s_full[1], 1);
        mbar_init(&sm.p_full, 256);
        mbar_init(&sm.pv_done, 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc_pair(&sm.tmem_base, 512);
    tc_fence_before();
    cluster_sync_all();  // barriers initialised in both CTAs before any remote arrival
    tc_fence_after();
    const uint32_t tmem = sm.tmem_base;
    const uint32_t t_lo = tmem + 256, t_o = tmem + 384;
    const int n_items = nkv * 8;

    if (warp == 0) {
        // ---------------------------------------------------------------- TMA (both CTAs)
        if (lane == 0) {
            mbar_arrive_expect_tx(&sm.q_full, 4 * CHUNK_BYTES);
            for (int c = 0; c < 4; ++c) tma_load_3d(sm.q_hi[c], &tm_q, &sm.q_full, 32 * c, t * TBM, h);
            int it = 0;
            auto load = [&](int j, bool is_v) {
                for (int c = 0; c < 4; ++c, ++it) {
                    const int s = it % NSTG2;
                    if (it >= NSTG2) mbar_wait(&sm.empty[s], ((it / NSTG2) - 1) & 1);
                    mbar_arrive_expect_tx(&sm.raw_full[s], HALF_BYTES);
                    if (!is_v) {  // keys [64 rank, +64) of tile j, dims [32 c, +32)
                        tma_load_3d(sm.hi[s], &tm_k, &sm.raw_full[s], 32 * c, j * TBM + 64 * (int)rank, kvh);
                    } else {  // keys [32 c, +32) of tile j, dims [64 rank, +64): two N atoms
                        for (int a = 0; a < 2; ++a)
                            tma_load_3d(sm.hi[s] + a * 4096, &tm_v, &sm.raw_full[s],
                                        64 * (int)rank + 32 * a, j * TBM + 32 * c, kvh);
                    }
                }
            };
            load(0, false);
            for (int j = 0; j < nkv; ++j) {
                if (j + 1 < nkv) load(j + 1, false);
                load(j, true);
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ---------------------------------------------------------------- MMA (leader)
        if (leader) {
            const uint32_t issue = elect_one() ? 1u : 0u;
            constexpr uint32_t id_s = idesc_tf32(0, 256), id_pv = idesc_tf32(1, 256);
            mbar_wait_cluster(&sm.q_ready, 0);
            tc_fence_after();
            int it = 0;
            auto issue_s = [&](int j) {
                const uint32_t t_s = tmem + 128 * (j & 1);
                for (int c = 0; c < 4; ++c, ++it) {
                    const int s = it % NSTG2;
                    mbar_wait_cluster(&sm.conv_full[s], (it / NSTG2) & 1);
                    tc_fence_after();
                    const uint32_t qh = smem_u32(sm.q_hi[c]), ql = smem_u32(sm.q_lo[c]);
                    const uint32_t kh = smem_u32(sm.hi[s]), kl = smem_u32(sm.lo[s]);
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        const uint32_t off = kk * 32;
                        mma_tf32_ss_pair_p(t_s, kdesc(qh + off), kdesc(kh + off), id_s, (c | kk) ? 1u : 0u, issue);
                        mma_tf32_ss_pair_p(t_s, kdesc(qh + off), kdesc(kl + off), id_s, 1u, issue);
                        mma_tf32_ss_pair_p(t_s, kdesc(ql + off), kdesc(kh + off), id_s, 1u, issue);
                    }
                    mma_commit_pair_p(&sm.empty[s], issue);
                }
                mma_commit_pair_p(&sm.s_full[j & 1], issue);
            };
            issue_s(0);
            for (int j = 0; j < nkv; ++j) {
                if (j + 1 < nkv) issue_s(j + 1);
                mbar_wait_cluster(&sm.p_full, j & 1);
                tc_fence_after();
                const uint32_t t_p = tmem + 128 * (j & 1);
                for (int c = 0; c < 4; ++c, ++it) {
                    const int s = it % NSTG2;
                    mbar_wait_cluster(&sm.conv_full[s], (it / NSTG2) & 1);
                    tc_fence_after();
                    const uint32_t vh = smem_u32(sm.hi[s]), vl = smem_u32(sm.lo[s]);
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        const uint32_t col = c * 32 + kk * 8, off = kk * 1024;
                        mma_tf32_ts_pair_p(t_o, t_p + col, ndesc(vh + off), id_pv, (j | c | kk) ? 1u : 0u, issue);
                        mma_tf32_ts_pair_p(t_o, t_p + col, ndesc(vl + off), id_pv, 1u, issue);
                        mma_tf32_ts_pair_p(t_o, t_lo + col, ndesc(vh + off), id_pv, 1u, issue);
                    }
                    mma_commit_pair_p(&sm.empty[s], issue);
                }
                mma_commit_pair_p(&sm.pv_done, issue);
            }
        }
    } else if (warp < 6) {
        // ---------------------------------------------------------------- split (both CTAs)
        const uint32_t tid = threadIdx.x - 64;
        mbar_wait(&sm.q_full, 0);
        for (int c = 0; c < 4; ++c) split_chunk(sm.q_hi[c], sm.q_lo[c], tid);
        fence_proxy_async_smem();
        mbar_arrive_leader_release(&sm.q_ready);
        for (int it = 0; it < n_items; ++it) {
            const int s = it % NSTG2;
            mbar_wait(&sm.raw_full[s], (it / NSTG2) & 1);
            split_chunk<HALF_BYTES>(sm.hi[s], sm.lo[s], tid);
            fence_proxy_async_smem();
            mbar_arrive_leader_release(&sm.conv_full[s]);
        }
    } else {
        // ---------------------------------------------------------------- softmax (both CTAs)
        const uint32_t quarter = warp & 3;
        const int row = t * TBM + (int)(quarter * 32 + lane);
        const uint32_t lane_off = (quarter * 32) << 16;
        float m = -INFINITY, l = 0.0f;
        for (int j = 0; j < nkv; ++j) {
            const uint32_t t_s = tmem + 128 * (j & 1);
            mbar_wait(&sm.s_full[j & 1], (j >> 1) & 1);
            tc_fence_after();
            const bool masked = j >= t;  // the diagonal tile, or (lower tile) the one past it
            float mx = -INFINITY;
#pragma unroll 1
            for (int c = 0; c < 4; ++c) {
                uint32_t r[32];
                tmem_ld32(t_s + lane_off + c * 32, r);
                tmem_wait_ld();
#pragma unroll
                for (int e = 0; e < 32; ++e) {
                    const int key = j * TBM + c * 32 + e;
                    const float x = __fmul_rn(__uint_as_float(r[e]), scale);
                    if (!masked || key <= row) mx = fmaxf(mx, x);
                }
            }
            if (j > 0) {
                mbar_wait(&sm.pv_done, (j - 1) & 1);
                tc_fence_after();
            }
            const float m_new = fmaxf(m, mx);
            const float corr = (m == -INFINITY) ? 0.0f : ex2_approx(__fmul_rn(m - m_new, kLog2e));
            if (j > 0 && __any_sync(0xffffffffu, corr != 1.0f)) {
#pragma unroll 1
                for (int c = 0; c < 4; ++c) {
                    uint32_t r[32];
                    tmem_ld32(t_o + lane_off + c * 32, r);
                    tmem_wait_ld();
#pragma unroll
                    for (int e = 0; e < 32; ++e) r[e] = __float_as_uint(__uint_as_float(r[e]) * corr);
                    tmem_st32(t_o + lane_off + c * 32, r);
                }
            }
            l *= corr;
            m = m_new;
#pragma unroll 1
            for (int c = 0; c < 4; ++c) {
                uint32_t r[32], rl[32];
                tmem_ld32(t_s + lane_off + c * 32, r);
                tmem_wait_ld();
#pragma unroll
                for (int e = 0; e < 32; ++e) {
                    const int key = j * TBM + c * 32 + e;
                    const float x = __fmul_rn(__uint_as_float(r[e]), scale);
                    const float pe = (!masked || key <= row) ? ex2_approx(__fmul_rn(x - m, kLog2e)) : 0.0f;
                    l += pe;
                    const float ph = tf32_hi(pe);
                    r[e] = __float_as_uint(ph);
                    rl[e] = __float_as_uint(pe - ph);
                }
                tmem_st32(t_s + lane_off + c * 32, r);
                tmem_st32(t_lo + lane_off + c * 32, rl);
            }
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive_leader_release(&sm.p_full);
        }
        mbar_wait(&sm.pv_done, (nkv - 1) & 1);
        tc_fence_after();
        const float inv_l = 1.0f / l;
        // o_rows: the decompress fused -- kept row `row` lands at its original position
        const int orow = (o_rows && row < n) ? __ldg(o_rows + (size_t)h * rows_per_head + row) : row;
        float* dst = o + ((size_t)h * rows_per_head + orow) * TD;
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
            uint32_t r[32];
            tmem_ld32(t_o + lane_off + c * 32, r);
            tmem_wait_ld();
            if (row < n) {
#pragma unroll
                for (int e = 0; e < 32; e += 4)
                    *reinterpret_cast<float4*>(dst + c * 32 + e) =
                        make_float4(__uint_as_float(r[e]) * inv_l, __uint_as_float(r[e + 1]) * inv_l,
                                    __uint_as_float(r[e + 2]) * inv_l, __uint_as_float(r[e + 3]) * inv_l);
            }
        }
    }
    tc_fence_before();
    cluster_sync_all();  // the leader's MMAs into this CTA's TMEM / smem are complete
    if (warp == 1) tmem_dealloc_pair(tmem, 512);
}

// 3-D [heads x rows x 128] f32, boxes of 32 x box_rows x 1 (128-B rows),
// swizzled for the operand's major-ness: rows past a head's end read zeros.
int make_f32_heads_map(CUtensorMap* m, const void* base, uint64_t rows, uint64_t heads,
                       uint32_t box_rows, CUtensorMapSwizzle swizzle) {
    auto fn = tensor_map_encoder();
    if (!fn) return invalid("tsa: cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[3] = {TD, rows, heads};
    cuuint64_t strides[2] = {TD * 4, rows * TD * 4};
    cuuint32_t box[3] = {32, box_rows, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, strides,
                    box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        return invalid("tsa: f32 tensor map encode failed (" + std::to_string((int)r) + ")");
    return 0;
}

}  // namespace

// The single-CTA kernel by default; TSA_TF32_PAIRS=1 selects the 2-CTA one
// (measured slower at cfg1: 237 vs 183 us under ncu, profiles/r2/ab_notes.txt;
// kept as the measured alternative and as a second implementation the tests
// compare against).
static bool tf32_pairs() {
    const char* e = getenv("TSA_TF32_PAIRS");
    return e && e[0] == '1';
}

bool attend_tf32_supported(const tsa_desc& d) { return d.dtype == TSA_F32 && d.d_head == TD; }

int launch_attend_tf32(const tsa_desc& d, const void* q, const void* k, const void* v,
                       const int32_t* n_dev, int32_t n_const, int32_t kv_group,
                       int32_t rows_per_head, int32_t kv_rows_per_head, void* o, cudaStream_t st,
                       const int32_t* o_rows) {
    if (!attend_tf32_supported(d)) return invalid("attend_tf32: needs f32, d_head 128");
    const int nh = d.head_end - d.head_begin;
    const int n_kv_buf = (d.n_heads + kv_group - 1) / kv_group;
    CUtensorMap mq, mk, mv;
    int rc;
    constexpr CUtensorMapSwizzle kK = CU_TENSOR_MAP_SWIZZLE_128B, kMN = CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B;
    const bool pair = tf32_pairs();
    if ((rc = make_f32_heads_map(&mq, q, rows_per_head, d.n_heads, 128, kK))) return rc;
    if ((rc = make_f32_heads_map(&mk, k, kv_rows_per_head, n_kv_buf, pair ? 64 : 128, kK))) return rc;
    if ((rc = make_f32_heads_map(&mv, v, kv_rows_per_head, n_kv_buf, 32, kMN))) return rc;
    const float scale = 1.0f / sqrtf((float)TD);
    if (pair) {
        const int smem = (int)sizeof(Tf32PairSmem) + 1024;
        if ((rc = ensure_smem_attr(reinterpret_cast<const void*>(attend_tf32_pair_kernel), smem)))
            return rc;
        const int max_pairs = ((rows_per_head + TBM - 1) / TBM + 1) / 2;
        dim3 grid(2 * nh, max_pairs);
        attend_tf32_pair_kernel<<<grid, kTf32Threads, smem, st>>>(
            mq, mk, mv, n_dev, n_const, kv_group, rows_per_head, d.head_begin, scale,
            static_cast<float*>(o), o_rows);
        TSA_LAUNCH_CHECK("attend_tf32_pair");
        return 0;
    }
    const int smem = (int)sizeof(Tf32Smem) + 1024;
    if ((rc = ensure_smem_attr(reinterpret_cast<const void*>(attend_tf32_kernel), smem))) return rc;
    dim3 grid(nh, (rows_per_head + TBM - 1) / TBM);
    attend_tf32_kernel<<<grid, kTf32Threads, smem, st>>>(mq, mk, mv, n_dev, n_const, kv_group,
                                                        rows_per_head, d.head_begin, scale,
                                                        static_cast<float*>(o), o_rows);
    TSA_LAUNCH_CHECK("attend_tf32");
    return 0;
}

}  // namespace tsa
