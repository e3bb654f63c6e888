// K1 EXACT: score_tokens (token_coverage.cpp:16-50) with the reference's f32
// arithmetic, bit for bit, at production speed (bf16 inputs, d = 128).
//
// The reference upcasts nothing -- it is f32 throughout -- so for bf16 inputs
// it computes, per query head h and tail row r (query L - lq + r):
//   X[r, j]  = (sum_p q[r,p] k[j,p], p ascending, f32, no FMA) * (1/sqrt d)
//                                              (tensor_ops.cpp:19-23, token_coverage.cpp:32-33)
//   m_r      = max over j <= L - lq + r        (tensor_ops.cpp:48-54)
//   e[r, j]  = expf(X[r, j] - m_r)             (glibc expf, :62)
//   sum_r    = e[r, 0] + e[r, 1] + ...         (sequential f32, :63)
//   P[r, j]  = e[r, j] / sum_r                 (:66-68)
//   c[j]     = P[0, j] + P[1, j] + ...         (r ascending, token_coverage.cpp:43-46)
//   s[h, t]  = avg_pool_1d(c, kernel)[t]       (tensor_ops.cpp:114-129)
// A bf16 x bf16 product has at most 16 significant bits, so q*k is exact in
// f32 and round(acc + round(q*k)) == fma(q, k, acc): the logits run as packed
// FFMA2 on the CUDA cores (the tensor cores' f32 accumulation does not round
// per addition, so it cannot reproduce the sequential order).  expf is
// glibc's algorithm ported bit for bit (expf_glibc.cuh).  Four launches:
//
//   score_exact_logits (XA): persistent, one CTA per SM over (KV group row
//     tile, 64-key tile) units.  The group's g*lq tail rows (up to 256) sit in
//     shared memory as f32; K tiles stream in by TMA (SW128, 4 stages); a
//     thread owns 8 rows x 8 keys and accumulates p = 0..127 in order (FFMA2,
//     the q value broadcast into both halves).  Writes X (f32, row stride
//     Lp = round_up(L, 64)) and the row maxima (order-independent, atomicMax
//     on an ordered-int encoding).  34.4 G FMA at 128K / Llama-3-8B: the
//     FP32 pipe is the roofline.
//   score_exact_rowsum (XB): the sequential row sums, one CTA per ~n_rows/#SM
//     rows (16 once that reaches 8): X tiles arrive by TMA, 15 helper warps
//     (thread = key x half the rows) compute e -- once: it is written back over
//     X -- into a shared tile, one warp (lane = row, float4 loads) runs the f32
//     chain in key order (L dependent FADDs per row: 0.32 ms floor at 128K,
//     0.51 ms measured).
//   score_exact_colsum (XC): thread = key, P = e / sum_r (Markstein division)
//     accumulated over r in order -> raw column sums.
//   pool: the shared edge-clamped pool kernel (score.cu).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <climits>

#include "common.cuh"
#include "chain_sum.cuh"
#include "expf_glibc.cuh"
#include "sm100.cuh"

namespace tsa {

int make_bf16_map_2d(CUtensorMap* m, const void* base, uint64_t rows, uint32_t box_rows);
int make_f32_map_2d(CUtensorMap* m, const void* base, uint64_t inner, uint64_t rows,
                    uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_rows);

namespace {

using namespace tsa_dev;

// ------------------------------------------------------------------ XA
constexpr int XA_ROWS = 256;   // tail rows per row tile (8 warps x 4 row groups x 8 rows)
constexpr int XA_KEYS = 64;    // keys per stage
constexpr int XA_STAGES = 4;
constexpr int XA_QS = 132;     // f32 per Q row in shared memory (+4: conflict-free row groups)
constexpr int XA_THREADS = 256;
constexpr int XA_KTILE = XA_KEYS * 128 * 2;  // 16 KB: two SW128 halves (d 0..63, 64..127)
constexpr int XA_KHALF = XA_KTILE / 2;

struct __align__(1024) XaSmem {
    uint8_t k[XA_STAGES][XA_KTILE];
    alignas(16) float q[XA_ROWS * XA_QS];
    uint64_t full[XA_STAGES];
    uint64_t empty[XA_STAGES];
};


// bf16 halves of a word as f32, by byte permutes (ALU pipe: a shift or mask
// may be emitted as IMAD, which would take FMA-pipe slots from the FFMA2s)
__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(__byte_perm(w, 0u, 0x1044)); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(__byte_perm(w, 0u, 0x3244)); }

// Aligned view of dynamic shared memory that keeps the pointer derived from
// the __shared__ array, so accesses compile to LDS/STS (not generic LD/ST).
template <typename T, uint32_t kAlign>
__device__ __forceinline__ T& smem_view(uint8_t* raw) {
    const uint32_t a = smem_u32(raw);
    return *reinterpret_cast<T*>(raw + ((kAlign - (a & (kAlign - 1))) & (kAlign - 1)));
}
__device__ __forceinline__ uint32_t word(const uint4& v, int i) {
    return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}
struct RowGeom {
    int hl;  // head relative to the shard's first head
    int r;   // tail row
    bool valid;
};

__global__ void __launch_bounds__(XA_THREADS, 1)
score_exact_logits(const __grid_constant__ CUtensorMap tm_k, const __nv_bfloat16* __restrict__ q,
                   int L, int Lp, int lq, int group, int rows_grp, int rt_per_kv, int n_ktiles,
                   int n_units, float inv_sqrt_d, float* __restrict__ X, int* __restrict__ rowmax) {
    extern __shared__ uint8_t smem_raw[];
    XaSmem& sm = smem_view<XaSmem, 1024>(smem_raw);
    const int u0 = (int)((long long)blockIdx.x * n_units / gridDim.x);
    const int u1 = (int)((long long)(blockIdx.x + 1) * n_units / gridDim.x);
    const int n = u1 - u0;
    if (n <= 0) return;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int rg = lane >> 3, kg = lane & 7;
    if (tid == 0) {
        for (int s = 0; s < XA_STAGES; ++s) {
            mbar_init(&sm.full[s], 1);
            mbar_init(&sm.empty[s], XA_THREADS / 32);
        }
        fence_barrier_init();
    }
    __syncthreads();
    auto issue = [&](int i) {
        const int st = i % XA_STAGES;
        if (i >= XA_STAGES) mbar_wait(&sm.empty[st], ((i / XA_STAGES) - 1) & 1);
        const int u = u0 + i;
        const int kv = (u / n_ktiles) / rt_per_kv, kt = u % n_ktiles;
        const int row = kv * L + kt * XA_KEYS;
        mbar_arrive_expect_tx(&sm.full[st], XA_KTILE);
        tma_load_2d(sm.k[st], &tm_k, &sm.full[st], 0, row);
        tma_load_2d(sm.k[st] + XA_KHALF, &tm_k, &sm.full[st], 64, row);
    };
    if (tid == 0)
        for (int i = 0; i < min(n, XA_STAGES - 1); ++i) issue(i);

    int rt_cur = -1;
    RowGeom rows[8];
    float rmax[8];
    // this thread's tile rows: lr0 + 4 a (the 4 row groups of a warp read adjacent
    // rows: with the 132-float pitch their 16-B loads fall in distinct banks)
    const int lr0 = warp * 32 + rg;
    auto flush = [&]() {
#pragma unroll
        for (int a = 0; a < 8; ++a) {
            float m = rmax[a];
            m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 1));
            m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 2));
            m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 4));
            if (kg == 0 && rows[a].valid && m != -INFINITY)
                atomicMax(&rowmax[rows[a].hl * lq + rows[a].r], enc_max(m));
        }
    };

    for (int i = 0; i < n; ++i) {
        const int u = u0 + i;
        const int rt = u / n_ktiles, kt = u % n_ktiles;
        if (tid == 0 && i + XA_STAGES - 1 < n) issue(i + XA_STAGES - 1);
        if (rt != rt_cur) {
            if (rt_cur >= 0) flush();
            named_bar_sync(1, XA_THREADS);  // every warp is done with the previous rows
            const int kv = rt / rt_per_kv, sub = rt % rt_per_kv;
            // stage the tile's tail rows as f32 (zeros past the group's rows)
            for (int e = tid; e < XA_ROWS * 16; e += XA_THREADS) {
                const int lr = e >> 4, c = e & 15;
                const int gr = sub * XA_ROWS + lr;
                float4 lo = make_float4(0.f, 0.f, 0.f, 0.f), hi = lo;
                if (gr < rows_grp) {
                    const int h = kv * group + gr / lq, r = gr % lq;
                    const uint4 v = *reinterpret_cast<const uint4*>(
                        q + ((size_t)h * L + (L - lq + r)) * 128 + c * 8);
                    lo = make_float4(bf16_lo(v.x), bf16_hi(v.x), bf16_lo(v.y), bf16_hi(v.y));
                    hi = make_float4(bf16_lo(v.z), bf16_hi(v.z), bf16_lo(v.w), bf16_hi(v.w));
                }
                *reinterpret_cast<float4*>(&sm.q[lr * XA_QS + c * 8]) = lo;
                *reinterpret_cast<float4*>(&sm.q[lr * XA_QS + c * 8 + 4]) = hi;
            }
#pragma unroll
            for (int a = 0; a < 8; ++a) {
                const int gr = sub * XA_ROWS + lr0 + 4 * a;
                rows[a].valid = gr < rows_grp;
                rows[a].hl = kv * group + gr / lq;
                rows[a].r = gr % lq;
                rmax[a] = -INFINITY;
            }
            named_bar_sync(1, XA_THREADS);
            rt_cur = rt;
        }
        const int st = i % XA_STAGES;
        mbar_wait(&sm.full[st], (i / XA_STAGES) & 1);

        uint64_t acc[8][4];
#pragma unroll
        for (int a = 0; a < 8; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) acc[a][b] = 0ull;
        const uint8_t* kb = sm.k[st];
        const float* qb = &sm.q[lr0 * XA_QS];
        // 16 blocks of 8 d-columns.  K words (8 keys x 8 columns, 8 x LDS.128) and
        // Q values (8 rows x 2 columns, 8 x LDS.64) for the next block / column
        // pair are loaded one step ahead into a second register set, so the
        // FFMA2 stream does not wait on LDS latency with two warps per scheduler.
        // K chunk c of key (kg + 8 i) sits at SW128 position (c & 7) ^ kg:
        // base ^ ((c & 7) << 4) with the kg bits pre-set (tiles are 1 KB aligned).
        const uint32_t kbase = smem_u32(kb) + kg * 128 + (kg << 4);
        const uint32_t qbase = smem_u32(qb);
        auto kaddr = [&](int c) { return (kbase ^ ((c & 7) << 4)) + (c >> 3) * XA_KHALF; };
        auto lds128 = [](uint32_t a) {
            uint4 v;
            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
            return v;
        };
        auto lds64f = [](uint32_t a) {
            float2 v;
            asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a));
            return v;
        };
        auto load_k = [&](int c, uint4 (&kw)[8]) {
            const uint32_t a = kaddr(c);
#pragma unroll
            for (int i8 = 0; i8 < 8; ++i8) kw[i8] = lds128(a + i8 * 1024);
        };
        auto load_q = [&](int p2, float2 (&qv)[8]) {  // columns 2 p2, 2 p2 + 1
#pragma unroll
            for (int a = 0; a < 8; ++a) qv[a] = lds64f(qbase + (4 * a * XA_QS + 2 * p2) * 4);
        };
        auto fma_col = [&](const uint4 (&kw)[8], int p8, float q0, int a, uint64_t (&kp)[4]) {
            (void)kw; (void)p8;
            const uint64_t qq = f2(q0, q0);
#pragma unroll
            for (int i2 = 0; i2 < 4; ++i2) acc[a][i2] = fma2(qq, kp[i2], acc[a][i2]);
        };
        auto pairs = [&](const uint4 (&kw)[8], int p8, uint64_t (&kp)[4]) {  // column p8 of the block
#pragma unroll
            for (int i2 = 0; i2 < 4; ++i2) {
                const uint32_t w0 = word(kw[2 * i2], p8 >> 1), w1 = word(kw[2 * i2 + 1], p8 >> 1);
                kp[i2] = (p8 & 1) ? f2(bf16_hi(w0), bf16_hi(w1)) : f2(bf16_lo(w0), bf16_lo(w1));
            }
        };
        auto block = [&](const uint4 (&kw)[8], float2 (&qA)[8], float2 (&qB)[8], int c,
                         bool prefetch_next) {
            // columns 8c .. 8c+7 as 4 column pairs; q pair j+1 loads while pair j computes
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                float2 (&cur)[8] = (j & 1) ? qB : qA;
                float2 (&nxt)[8] = (j & 1) ? qA : qB;
                if (j < 3 || prefetch_next) load_q(4 * c + j + 1, nxt);
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    uint64_t kp[4];
                    pairs(kw, 2 * j + e, kp);
#pragma unroll
                    for (int a = 0; a < 8; ++a) fma_col(kw, 2 * j + e, e ? cur[a].y : cur[a].x, a, kp);
                }
            }
        };
        uint4 kwA[8], kwB[8];
        float2 qA[8], qB[8];
        load_k(0, kwA);
        load_q(0, qA);
#pragma unroll 1
        for (int c = 0; c < 16; c += 2) {
            load_k(c + 1, kwB);
            block(kwA, qA, qB, c, true);
            if (c + 2 < 16) load_k(c + 2, kwA);
            block(kwB, qA, qB, c + 1, c + 2 < 16);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.empty[st]);

        // epilogue: scale (f32 multiply after the dot, token_coverage.cpp:33), causal
        // mask, store X, running row max
        const int key0 = kt * XA_KEYS + kg;
#pragma unroll
        for (int a = 0; a < 8; ++a) {
            if (!rows[a].valid) continue;
            const int limit = L - lq + rows[a].r;
            float* xr = X + (size_t)(rows[a].hl * lq + rows[a].r) * Lp;
#pragma unroll
            for (int i2 = 0; i2 < 4; ++i2) {
                float x0, x1;
                f2_split(acc[a][i2], x0, x1);
                x0 = __fmul_rn(x0, inv_sqrt_d);
                x1 = __fmul_rn(x1, inv_sqrt_d);
                const int j0 = key0 + 16 * i2, j1 = j0 + 8;
                if (j0 <= limit) {
                    xr[j0] = x0;
                    rmax[a] = fmaxf(rmax[a], x0);
                }
                if (j1 <= limit) {
                    xr[j1] = x1;
                    rmax[a] = fmaxf(rmax[a], x1);
                }
            }
        }
    }
    flush();
}

// ------------------------------------------------------------------ XB
// Rows per CTA are chosen at run time (<= 16, one chain lane each) so the
// exponentials -- the bulk of this kernel's work -- spread over every SM.
constexpr int XB_MAXR = 16;
// 15 helper warps over 240-key tiles: warp 15 sums, on a sub-partition that holds
// three helpers instead of four (less issue competition for its dependent FADDs);
// 16 x 256, 12 x 192, 14 x 224, 11 x 176 and a sub-partition to itself all measured
// slower (profiles/r2/ab_notes.txt).  Build-time knobs for such A/B runs:
#ifndef TSA_XB_KEYS
#define TSA_XB_KEYS 240
#endif
#ifndef TSA_XB_HELP
#define TSA_XB_HELP 15
#endif
constexpr int XB_KEYS = TSA_XB_KEYS;
constexpr int XB_STAGES = 4;                      // e tiles in flight
constexpr int XB_XST = 8;                         // X tiles in flight (HBM latency x bandwidth)
constexpr int XB_HELP = TSA_XB_HELP;              // helper warps: thread = (key, part of the rows)
constexpr int XB_PARTS = XB_HELP * 32 / XB_KEYS;  // row parts per key column
constexpr int XB_CH = XB_KEYS % 32 == 0 ? 32 : 16;  // chain chunk (keys)
static_assert(XB_PARTS * XB_KEYS == XB_HELP * 32 && XB_MAXR % XB_PARTS == 0 && XB_KEYS % 16 == 0,
              "row-sum helper geometry");
constexpr int XB_THREADS = 32 * (XB_HELP + 1);    // + the summing warp
// e tile row pitch in floats: 4 (256 keys) or 20 (240) mod 32 makes the helpers' row
// stores (lane = key) and the summing warp's float4 loads (lane = row, 8 rows a
// wavefront) conflict-free
constexpr int XB_EP = XB_KEYS + 4;
// Rows per row-sum CTA (chain mode) at or below which the chains run apart
// (row_chain_sum) and the exponentials split over key ranges.
constexpr int kSplitRowsPerCta = 4;

struct __align__(128) XbSmem {
    float x[XB_XST][XB_MAXR * XB_KEYS];           // X tile (TMA), rows x keys
    alignas(16) float e[XB_STAGES][XB_MAXR * XB_EP];  // e tile, rows x keys
    uint64_t tab[32];                             // glibc's exp2f table
    float m[XB_MAXR];
    int allowed[XB_MAXR];
    uint64_t x_full[XB_XST], x_empty[XB_XST], e_full[XB_STAGES], e_empty[XB_STAGES];
};

// kChain = false: the exponentials only (e written over X); the row sums then
// come from row_chain_sum below (few rows: each CTA's L-long chain would be the
// whole kernel's floor).
template <bool kChain>
__global__ void __launch_bounds__(XB_THREADS, 1)
score_exact_rowsum(const __grid_constant__ CUtensorMap tm_x, float* __restrict__ X, int L, int Lp,
                   int lq, int n_rows, int rows_per_cta, int tiles_per_split,
                   const int* __restrict__ rowmax, float* __restrict__ rowsum) {
    extern __shared__ uint8_t smem_raw[];
    XbSmem& sm = smem_view<XbSmem, 128>(smem_raw);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int R = rows_per_cta;
    const int row0 = blockIdx.x * R;  // rows of X: (local head, r) flattened
    exp2f_table_to_smem(sm.tab);
    if (tid < XB_MAXR) {
        const int gr = row0 + tid;
        const bool ok = tid < R && gr < n_rows;
        sm.m[tid] = ok ? dec_max(rowmax[gr]) : 0.0f;
        sm.allowed[tid] = ok ? L - lq + gr % lq + 1 : 0;
    }
    if (tid == 0) {
        for (int s = 0; s < XB_XST; ++s) {
            mbar_init(&sm.x_full[s], 1);
            mbar_init(&sm.x_empty[s], XB_HELP);
        }
        for (int s = 0; s < XB_STAGES; ++s) {
            mbar_init(&sm.e_full[s], XB_HELP * 32);
            mbar_init(&sm.e_empty[s], 32);
        }
        fence_barrier_init();
    }
    __syncthreads();
    // this CTA's key tiles: all of them with the chain; a range of them (blockIdx.y)
    // for the exponentials alone
    const int tb = blockIdx.y * tiles_per_split;
    const int n_tiles = min((L + XB_KEYS - 1) / XB_KEYS - tb, tiles_per_split);
    auto issue = [&](int t) {  // t: local tile index
        const int st = t % XB_XST;
        if (t >= XB_XST) mbar_wait(&sm.x_empty[st], ((t / XB_XST) - 1) & 1);
        mbar_arrive_expect_tx(&sm.x_full[st], R * XB_KEYS * 4);
        tma_load_2d(sm.x[st], &tm_x, &sm.x_full[st], (tb + t) * XB_KEYS, row0);
    };
    if (warp < XB_HELP) {
        if (tid == 0)
            for (int t = 0; t < min(n_tiles, XB_XST - 1); ++t) issue(t);
        // thread = key column j of the tile: XB_MAXR independent exponentials per
        // tile, unconditionally (rows >= R are padding the chain never reads), so
        // they interleave
        constexpr int RH = XB_MAXR / XB_PARTS;
        const int j = tid % XB_KEYS, rbase = (tid / XB_KEYS) * RH;
        float mrow[RH];
        int arow[RH];
#pragma unroll
        for (int i = 0; i < RH; ++i) {
            mrow[i] = sm.m[rbase + i];
            arow[i] = sm.allowed[rbase + i];
        }
        const bool full_rows = R == XB_MAXR && row0 + XB_MAXR <= n_rows;
        for (int t = 0; t < n_tiles; ++t) {
            if (tid == 0 && t + XB_XST - 1 < n_tiles) issue(t + XB_XST - 1);
            const int xt = t % XB_XST, st = t % XB_STAGES;
            mbar_wait(&sm.x_full[xt], (t / XB_XST) & 1);
            if (kChain && t >= XB_STAGES) mbar_wait(&sm.e_empty[st], ((t / XB_STAGES) - 1) & 1);
            const float* xs = sm.x[xt] + rbase * XB_KEYS + j;
            float* es = sm.e[st] + rbase * XB_EP + j;
            const int key = (tb + t) * XB_KEYS + j;
            float xv[RH];
#pragma unroll
            for (int i = 0; i < RH; ++i) xv[i] = xs[i * XB_KEYS];
            // e overwrites X in HBM (the column pass reads it: the exponentials run once)
            float* xg = X + (size_t)(row0 + rbase) * Lp + key;
            // (CTA-uniform) every row live and no key of the tile past any row's causal
            // limit: no per-element mask
            if (full_rows && (tb + t + 1) * XB_KEYS <= L - lq + 1) {
#pragma unroll
                for (int i = 0; i < RH; ++i) {
                    const float e = expf_glibc(__fsub_rn(xv[i], mrow[i]), sm.tab);
                    if (kChain) es[i * XB_EP] = e;
                    __stcs(xg + (size_t)i * Lp, e);
                }
            } else if (rbase < R)  // (warp-uniform) a half with no live rows skips its exponentials
#pragma unroll
            for (int i = 0; i < RH; ++i) {
                // masked entries add +0 to the chain: exactly the reference's skip
                const float e = expf_glibc(__fsub_rn(xv[i], mrow[i]), sm.tab);
                const bool ok = key < arow[i];
                if (kChain) es[i * XB_EP] = ok ? e : 0.0f;
                if (ok) __stcs(xg + (size_t)i * Lp, e);
            }
            // every helper thread publishes its own e writes (release) to the chain warp
            if (kChain) mbar_arrive(&sm.e_full[st]);
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.x_empty[xt]);
        }
    } else if (kChain) {
        // the sequential f32 row sums, lane = row (tensor_ops.cpp:59-65)
        const int row = lane & (XB_MAXR - 1);
        float s = 0.0f;
        for (int t = 0; t < n_tiles; ++t) {
            const int st = t % XB_STAGES;
            mbar_wait(&sm.e_full[st], (t / XB_STAGES) & 1);
            // the row's keys as float4 (one LDS.128 per 4 FADDs); the next 32
            // values load while the current 32 are added (off the FADD chain)
            const float4* es = reinterpret_cast<const float4*>(sm.e[st] + row * XB_EP);
            constexpr int V = XB_CH / 4;
            float4 cur[V], nxt[V];
#pragma unroll
            for (int i = 0; i < V; ++i) cur[i] = es[i];
#pragma unroll
            for (int c = 0; c < XB_KEYS / XB_CH; ++c) {
                if (c + 1 < XB_KEYS / XB_CH) {
#pragma unroll
                    for (int i = 0; i < V; ++i) nxt[i] = es[(c + 1) * V + i];
                }
#pragma unroll
                for (int i = 0; i < V; ++i) {
                    s = __fadd_rn(s, cur[i].x);
                    s = __fadd_rn(s, cur[i].y);
                    s = __fadd_rn(s, cur[i].z);
                    s = __fadd_rn(s, cur[i].w);
                }
#pragma unroll
                for (int i = 0; i < V; ++i) cur[i] = nxt[i];
            }
            mbar_arrive(&sm.e_empty[st]);  // each lane's reads of the stage are done
        }
        if (lane < R && row0 + lane < n_rows) rowsum[row0 + lane] = s;
    }
}

// The row sums of few rows: one CTA per row, the exact sequential f32 sum of
// its e values (the first L - lq + r + 1 keys; the masked tail adds nothing)
// without the L-long chain (chain_sum.cuh).
constexpr int XR_THREADS = 512;
__global__ void __launch_bounds__(XR_THREADS) row_chain_sum(const float* __restrict__ X, int L, int Lp,
                                                            int lq, float* __restrict__ rowsum) {
    const int row = blockIdx.x;
    const int n = min(L, L - lq + row % lq + 1);
    const float s = exact_chain_sum<XR_THREADS>(X + (size_t)row * Lp, n);
    if (threadIdx.x == 0) rowsum[row] = s;
}

__global__ void fill_int(int* __restrict__ p, int v, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

// ------------------------------------------------------------------ XC
constexpr int XC_KEYS = 128;   // keys per CTA (thread = key)
constexpr int XC_ROWS = 64;    // rows per TMA chunk
constexpr int XC_STAGES = 2;

// e / sum, correctly rounded, from y = RN(1/sum): q = RN(e y), r = e - q sum
// (exact, FMA), RN(q + r y) = RN(e / sum) (Markstein) -- valid while the
// quotient is normal (e >= 2^-100 > 2^-126 * sum for sum <= 2^26).  Below
// that: e = 0 gives 0, and a tiny e is divided in double and rounded once more
// to f32 -- exact, as double rounding is innocuous for a quotient computed with
// at least 2 * 24 + 2 bits (sharp maps have many such e: __fdiv_rn's slow path
// made the column pass 4x slower on cfg4's layers).
__device__ __forceinline__ float div_rn(float e, float sum, float y) {
    if (e >= 0x1p-100f) {
        const float q = __fmul_rn(e, y);
        const float r = __fmaf_rn(-q, sum, e);
        return __fmaf_rn(r, y, q);
    }
    if (e == 0.0f) return 0.0f;
    return __double2float_rn(__ddiv_rn((double)e, (double)sum));
}

// shared memory: [XcHead][rs: lq x float4][n_st x X chunk (32 KB)]
struct __align__(128) XcHead {
    uint64_t tab[32];
    uint64_t full[XC_STAGES];
};
__host__ __device__ constexpr int xc_rs_bytes(int lq) { return (lq * 16 + 127) / 128 * 128; }

// c[j] = sum over r (ascending) of e[r, j] / sum_r, reading the e rows the
// row-sum pass wrote over X; chunks [64 rows x 128 keys] arrive by TMA, so
// many loads are in flight without registers.
__global__ void __launch_bounds__(XC_KEYS)
score_exact_colsum(const __grid_constant__ CUtensorMap tm_x, int L, int lq, int head_begin,
                   const int* __restrict__ rowmax, const float* __restrict__ rowsum,
                   float* __restrict__ colraw) {
    extern __shared__ uint8_t smem_raw[];
    XcHead& sm = smem_view<XcHead, 128>(smem_raw);
    float4* rs = reinterpret_cast<float4*>(&sm + 1);  // per row: -, sum, RN(1/sum)
    float* xbuf = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(rs) + xc_rs_bytes(lq));
    const int tid = threadIdx.x;
    const int hl = blockIdx.y;
    const int k0 = blockIdx.x * XC_KEYS;
    (void)rowmax;
    const int n_chunks = (lq + XC_ROWS - 1) / XC_ROWS;
    const int n_st = min(n_chunks, XC_STAGES);
    const int row_base = hl * lq;
    if (tid == 0) {
        for (int s = 0; s < XC_STAGES; ++s) mbar_init(&sm.full[s], 1);
        fence_barrier_init();
        for (int c = 0; c < n_st; ++c) {
            mbar_arrive_expect_tx(&sm.full[c], XC_ROWS * XC_KEYS * 4);
            tma_load_2d(xbuf + c * XC_ROWS * XC_KEYS, &tm_x, &sm.full[c], k0, row_base + c * XC_ROWS);
        }
    }
    for (int r = tid; r < lq; r += XC_KEYS) {
        const float sum = rowsum[row_base + r];
        rs[r] = make_float4(0.0f, sum, __frcp_rn(sum), 0.0f);
    }
    __syncthreads();
    const int j = k0 + tid;
    // row r sees key j iff j <= L - lq + r (token_coverage.cpp:36-41)
    const int r_first = max(0, j - (L - lq));
    float c = 0.0f;
    for (int ch = 0; ch < n_chunks; ++ch) {
        const int st = ch % n_st;
        mbar_wait(&sm.full[st], (ch / n_st) & 1);
        const float* xs = xbuf + st * XC_ROWS * XC_KEYS + tid;
        const int r0 = ch * XC_ROWS;
        const int rn = min(XC_ROWS, lq - r0);
        if (r_first <= r0 && rn == XC_ROWS) {  // every row of the chunk sees the key
#pragma unroll 16
            for (int i = 0; i < XC_ROWS; ++i) {
                const float4 w = rs[r0 + i];
                c = __fadd_rn(c, div_rn(xs[i * XC_KEYS], w.y, w.z));
            }
        } else {
            for (int i = max(0, r_first - r0); i < rn; ++i) {
                const float4 w = rs[r0 + i];
                c = __fadd_rn(c, div_rn(xs[i * XC_KEYS], w.y, w.z));
            }
        }
        __syncthreads();  // the stage is refilled below
        if (tid == 0 && ch + n_st < n_chunks) {
            mbar_arrive_expect_tx(&sm.full[st], XC_ROWS * XC_KEYS * 4);
            tma_load_2d(xbuf + st * XC_ROWS * XC_KEYS, &tm_x, &sm.full[st], k0,
                        row_base + (ch + n_st) * XC_ROWS);
        }
    }
    if (j < L) colraw[(size_t)(head_begin + hl) * L + j] = c;
}

__global__ void expf_kernel(const float* __restrict__ x, float* __restrict__ y, int64_t n) {
    __shared__ uint64_t tab[32];
    exp2f_table_to_smem(tab);
    __syncthreads();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        y[i] = expf_glibc(x[i], tab);
}

}  // namespace

int launch_expf(const float* x, float* y, int64_t n, cudaStream_t st) {
    if (n <= 0) return 0;
    const int grid = (int)std::min<int64_t>((n + 255) / 256, 8 * num_sms());
    expf_kernel<<<grid, 256, 0, st>>>(x, y, n);
    TSA_LAUNCH_CHECK("expf");
    return 0;
}

bool score_exact_supported(const tsa_desc& d) { return d.dtype == TSA_BF16 && d.d_head == 128; }

size_t exact_logits_stride(int L) { return align_up((size_t)L, 64); }

int launch_score_exact(const tsa_desc& d, const void* q, const void* k, const OutReplicas& s,
                       float* X, int* rowmax, float* rowsum, float* colraw, cudaStream_t st) {
    if (!score_exact_supported(d)) return invalid("score_tokens: EXACT scoring needs bf16, d_head 128");
    const int L = d.seq_len, lq = lq_of(d);
    const int Lp = (int)exact_logits_stride(L);
    const int g = d.n_heads / d.n_kv_heads;
    const int kv_begin = d.head_begin / g, kv_end = d.head_end / g;
    const int n_kv = kv_end - kv_begin;
    const int nh = d.head_end - d.head_begin;
    const int rows_grp = g * lq;
    const int rt_per_kv = (rows_grp + XA_ROWS - 1) / XA_ROWS;
    const int n_ktiles = (L + XA_KEYS - 1) / XA_KEYS;
    const int n_units = n_kv * rt_per_kv * n_ktiles;
    const size_t eb = 2;
    const uint8_t* qb = static_cast<const uint8_t*>(q) + (size_t)kv_begin * g * L * 128 * eb;
    const uint8_t* kb = static_cast<const uint8_t*>(k) + (size_t)kv_begin * L * 128 * eb;
    CUtensorMap mk;
    int rc;
    if ((rc = make_bf16_map_2d(&mk, kb, (uint64_t)n_kv * L, XA_KEYS))) return rc;
    const int n_rows = nh * lq;
    const int nsm = num_sms();
    fill_int<<<(n_rows + 255) / 256, 256, 0, st>>>(rowmax, INT_MIN, n_rows);  // below every encoding
    TSA_LAUNCH_CHECK("score_exact_fill");
    {
        const int smem = (int)sizeof(XaSmem) + 1024;
        if ((rc = ensure_smem_attr(reinterpret_cast<const void*>(score_exact_logits), smem))) return rc;
        const int grid = std::max(1, std::min(nsm, n_units));
        const float inv_sqrt_d = 1.0f / sqrtf(128.0f);
        score_exact_logits<<<grid, XA_THREADS, smem, st>>>(
            mk, reinterpret_cast<const __nv_bfloat16*>(qb), L, Lp, lq, g, rows_grp, rt_per_kv,
            n_ktiles, n_units, inv_sqrt_d, X, rowmax);
        TSA_LAUNCH_CHECK("score_exact_logits");
    }
    return launch_score_exact_rows(d, X, rowmax, rowsum, colraw, s, st);
}

int launch_fill_int(int* p, int v, int n, cudaStream_t st) {
    fill_int<<<(n + 255) / 256, 256, 0, st>>>(p, v, n);
    TSA_LAUNCH_CHECK("fill_int");
    return 0;
}

int launch_score_exact_rows(const tsa_desc& d, float* X, int* rowmax, float* rowsum, float* colraw,
                            const OutReplicas& s, cudaStream_t st) {
    const int L = d.seq_len, lq = lq_of(d);
    const int Lp = (int)exact_logits_stride(L);
    const int nh = d.head_end - d.head_begin;
    const int n_rows = nh * lq;
    const int nsm = num_sms();
    // rows per row-sum CTA: spread the rows over every SM (<= 16: one chain lane each)
    // full 16-row CTAs once the rows reach 8 per SM (the chain length, not the CTA
    // count, sets the time; full CTAs take the unmasked tile path)
    const int rpc0 = std::max(1, (n_rows + nsm - 1) / nsm);
    const int rpc = rpc0 >= 8 ? XB_MAXR : std::min(XB_MAXR, rpc0);
    CUtensorMap mx;
    int rc;
    if ((rc = make_f32_map_2d(&mx, X, (uint64_t)Lp, (uint64_t)n_rows, (uint64_t)Lp * 4, XB_KEYS,
                              (uint32_t)rpc)))
        return rc;
    {
        // few rows (a head shard of a multi-GPU layer): the exponentials of full
        // 16-row CTAs split over key ranges, then the chain-free row sums;
        // otherwise each CTA's chains overlap its exponentials
        const bool split = rpc <= kSplitRowsPerCta;
        const int smem = (int)sizeof(XbSmem) + 128;
        const int n_tiles = (L + XB_KEYS - 1) / XB_KEYS;
        const int rows = split ? std::min(XB_MAXR, n_rows) : rpc;
        const int row_ctas = (n_rows + rows - 1) / rows;
        const int splits = split ? std::max(1, std::min(n_tiles, nsm / row_ctas)) : 1;  // one wave
        const int tps = (n_tiles + splits - 1) / splits;
        if (split && (rc = make_f32_map_2d(&mx, X, (uint64_t)Lp, (uint64_t)n_rows, (uint64_t)Lp * 4,
                                           XB_KEYS, (uint32_t)rows)))
            return rc;
        auto kern = split ? score_exact_rowsum<false> : score_exact_rowsum<true>;
        if ((rc = ensure_smem_attr(reinterpret_cast<const void*>(kern), smem))) return rc;
        kern<<<dim3(row_ctas, (n_tiles + tps - 1) / tps), XB_THREADS, smem, st>>>(
            mx, X, L, Lp, lq, n_rows, rows, tps, rowmax, rowsum);
        TSA_LAUNCH_CHECK("score_exact_rowsum");
        if (split) {
            row_chain_sum<<<n_rows, XR_THREADS, 0, st>>>(X, L, Lp, lq, rowsum);
            TSA_LAUNCH_CHECK("row_chain_sum");
        }
    }
    {
        CUtensorMap mxc;
        if ((rc = make_f32_map_2d(&mxc, X, (uint64_t)Lp, (uint64_t)n_rows, (uint64_t)Lp * 4,
                                  XC_KEYS, XC_ROWS)))
            return rc;
        const int n_st = std::min((lq + XC_ROWS - 1) / XC_ROWS, XC_STAGES);
        const int smem = (int)sizeof(XcHead) + 128 + xc_rs_bytes(lq) + n_st * XC_ROWS * XC_KEYS * 4;
        if ((rc = ensure_smem_attr(reinterpret_cast<const void*>(score_exact_colsum), smem))) return rc;
        dim3 grid((L + XC_KEYS - 1) / XC_KEYS, nh);
        score_exact_colsum<<<grid, XC_KEYS, smem, st>>>(mxc, L, lq, d.head_begin, rowmax, rowsum,
                                                         colraw);
        TSA_LAUNCH_CHECK("score_exact_colsum");
    }
    tsa_desc pd = d;
    pd.last_q = 1;
    return launch_colsum_pool(pd, colraw, s, st);
}

}  // namespace tsa
