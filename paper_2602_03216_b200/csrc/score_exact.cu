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
//   score_exact_rowsum (XB): the sequential row sums, one CTA per 16 rows: X
//     tiles arrive by TMA, 8 helper warps compute e into a transposed shared
//     tile, one warp (lane = row) runs the f32 chain in key order.  The chain
//     (L dependent FADDs per row) is this kernel's critical path.
//   score_exact_colsum (XC): thread = key, P = e / sum_r accumulated over r in
//     order -> raw column sums.
//   pool: the shared edge-clamped pool kernel (score.cu).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <climits>

#include "common.cuh"
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

__device__ __forceinline__ int enc_max(float f) {
    const int i = __float_as_int(f);
    return i >= 0 ? i : i ^ 0x7fffffff;
}
__device__ __forceinline__ float dec_max(int i) { return __int_as_float(i >= 0 ? i : i ^ 0x7fffffff); }

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
__device__ __forceinline__ float comp(const float4& v, int i) {
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
#pragma unroll 1
        for (int c = 0; c < 16; ++c) {
            // keys kg + 8 i, d columns c*8 .. c*8+7: SW128 chunk (c & 7) ^ (key & 7) = (c & 7) ^ kg
            const uint8_t* kc = kb + (c >> 3) * XA_KHALF + kg * 128 + (((c & 7) ^ kg) << 4);
            uint4 kw[8];
#pragma unroll
            for (int i8 = 0; i8 < 8; ++i8) kw[i8] = *reinterpret_cast<const uint4*>(kc + i8 * 1024);
#pragma unroll
            for (int sub = 0; sub < 2; ++sub) {
                float4 qv[8];
#pragma unroll
                for (int a = 0; a < 8; ++a)
                    qv[a] = *reinterpret_cast<const float4*>(qb + 4 * a * XA_QS + c * 8 + sub * 4);
#pragma unroll
                for (int pp = 0; pp < 4; ++pp) {
                    const int wi = sub * 2 + (pp >> 1);
                    uint64_t kp[4];  // key pairs (kg + 16 i2, kg + 16 i2 + 8)
#pragma unroll
                    for (int i2 = 0; i2 < 4; ++i2) {
                        const uint32_t w0 = word(kw[2 * i2], wi), w1 = word(kw[2 * i2 + 1], wi);
                        kp[i2] = (pp & 1) ? f2(bf16_hi(w0), bf16_hi(w1)) : f2(bf16_lo(w0), bf16_lo(w1));
                    }
#pragma unroll
                    for (int a = 0; a < 8; ++a) {
                        const float qs = comp(qv[a], pp);
                        const uint64_t qq = f2(qs, qs);
#pragma unroll
                        for (int i2 = 0; i2 < 4; ++i2) acc[a][i2] = fma2(qq, kp[i2], acc[a][i2]);
                    }
                }
            }
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
constexpr int XB_ROWS = 16;
constexpr int XB_KEYS = 256;
constexpr int XB_STAGES = 4;
constexpr int XB_HELP = 8;                        // helper warps (2 rows each)
constexpr int XB_THREADS = 32 * (XB_HELP + 1);    // + the summing warp
constexpr int XB_EP = XB_ROWS + 1;                // e tile row pitch (conflict-free transpose)

struct __align__(128) XbSmem {
    float x[XB_STAGES][XB_ROWS * XB_KEYS];
    float e[XB_STAGES][XB_KEYS * XB_EP];
    float m[XB_ROWS];
    int allowed[XB_ROWS];
    uint64_t x_full[XB_STAGES], x_empty[XB_STAGES], e_full[XB_STAGES], e_empty[XB_STAGES];
};

__global__ void __launch_bounds__(XB_THREADS, 1)
score_exact_rowsum(const __grid_constant__ CUtensorMap tm_x, int L, int lq, int n_rows,
                   const int* __restrict__ rowmax, float* __restrict__ rowsum) {
    extern __shared__ uint8_t smem_raw[];
    XbSmem& sm = smem_view<XbSmem, 128>(smem_raw);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int row0 = blockIdx.x * XB_ROWS;  // rows of X: (local head, r) flattened
    if (tid < XB_ROWS) {
        const int gr = row0 + tid;
        const bool ok = gr < n_rows;
        sm.m[tid] = ok ? dec_max(rowmax[gr]) : 0.0f;
        sm.allowed[tid] = ok ? L - lq + gr % lq + 1 : 0;
    }
    if (tid == 0) {
        for (int s = 0; s < XB_STAGES; ++s) {
            mbar_init(&sm.x_full[s], 1);
            mbar_init(&sm.x_empty[s], XB_HELP);
            mbar_init(&sm.e_full[s], XB_HELP);
            mbar_init(&sm.e_empty[s], 1);
        }
        fence_barrier_init();
    }
    __syncthreads();
    const int n_tiles = (L + XB_KEYS - 1) / XB_KEYS;
    auto issue = [&](int t) {
        const int st = t % XB_STAGES;
        if (t >= XB_STAGES) mbar_wait(&sm.x_empty[st], ((t / XB_STAGES) - 1) & 1);
        mbar_arrive_expect_tx(&sm.x_full[st], XB_ROWS * XB_KEYS * 4);
        tma_load_2d(sm.x[st], &tm_x, &sm.x_full[st], t * XB_KEYS, row0);
    };
    if (warp < XB_HELP) {
        if (tid == 0)
            for (int t = 0; t < min(n_tiles, XB_STAGES - 1); ++t) issue(t);
        const int ra = warp * 2;
        for (int t = 0; t < n_tiles; ++t) {
            if (tid == 0 && t + XB_STAGES - 1 < n_tiles) issue(t + XB_STAGES - 1);
            const int st = t % XB_STAGES;
            mbar_wait(&sm.x_full[st], (t / XB_STAGES) & 1);
            if (t >= XB_STAGES) mbar_wait(&sm.e_empty[st], ((t / XB_STAGES) - 1) & 1);
            const float* xs = sm.x[st];
            float* es = sm.e[st];
#pragma unroll
            for (int rr = 0; rr < 2; ++rr) {
                const int row = ra + rr;
                const float m = sm.m[row];
                const int allowed = sm.allowed[row];
#pragma unroll
                for (int e8 = 0; e8 < XB_KEYS / 32; ++e8) {
                    const int j = lane + 32 * e8;
                    const float x = xs[row * XB_KEYS + j];
                    // masked entries add +0 to the chain: exactly the reference's skip
                    const float v = t * XB_KEYS + j < allowed ? expf_glibc(__fsub_rn(x, m)) : 0.0f;
                    es[j * XB_EP + row] = v;
                }
            }
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&sm.x_empty[st]);
                mbar_arrive(&sm.e_full[st]);
            }
        }
    } else {
        // the sequential f32 row sums, lane = row (tensor_ops.cpp:59-65)
        const int row = lane & (XB_ROWS - 1);
        float s = 0.0f;
        for (int t = 0; t < n_tiles; ++t) {
            const int st = t % XB_STAGES;
            mbar_wait(&sm.e_full[st], (t / XB_STAGES) & 1);
            const float* es = sm.e[st] + row;
#pragma unroll 16
            for (int j = 0; j < XB_KEYS; ++j) s = __fadd_rn(s, es[j * XB_EP]);
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.e_empty[st]);
        }
        if (lane < XB_ROWS && row0 + lane < n_rows) rowsum[row0 + lane] = s;
    }
}

__global__ void fill_int(int* __restrict__ p, int v, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

// ------------------------------------------------------------------ XC
constexpr int XC_T = 256;

__global__ void __launch_bounds__(XC_T)
score_exact_colsum(const float* __restrict__ X, int L, int Lp, int lq, int head_begin,
                   const int* __restrict__ rowmax, const float* __restrict__ rowsum,
                   float* __restrict__ colraw) {
    extern __shared__ float st[];  // m[lq], sum[lq]
    const int hl = blockIdx.y;
    for (int r = threadIdx.x; r < lq; r += XC_T) {
        st[r] = dec_max(rowmax[hl * lq + r]);
        st[lq + r] = rowsum[hl * lq + r];
    }
    __syncthreads();
    const int j = blockIdx.x * XC_T + threadIdx.x;
    if (j >= L) return;
    const float* x = X + (size_t)hl * lq * Lp + j;
    // row r sees key j iff j <= L - lq + r (token_coverage.cpp:36-41)
    const int r_first = max(0, j - (L - lq));
    float c = 0.0f;
#pragma unroll 8
    for (int r = r_first; r < lq; ++r) {
        const float e = expf_glibc(__fsub_rn(x[(size_t)r * Lp], st[r]));
        c = __fadd_rn(c, __fdiv_rn(e, st[lq + r]));
    }
    colraw[(size_t)(head_begin + hl) * L + j] = c;
}

__global__ void expf_kernel(const float* __restrict__ x, float* __restrict__ y, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        y[i] = expf_glibc(x[i]);
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
    CUtensorMap mk, mx;
    int rc;
    if ((rc = make_bf16_map_2d(&mk, kb, (uint64_t)n_kv * L, XA_KEYS))) return rc;
    const int n_rows = nh * lq;
    if ((rc = make_f32_map_2d(&mx, X, (uint64_t)Lp, (uint64_t)n_rows, (uint64_t)Lp * 4, XB_KEYS,
                              XB_ROWS)))
        return rc;
    fill_int<<<(n_rows + 255) / 256, 256, 0, st>>>(rowmax, INT_MIN, n_rows);  // below every encoding
    TSA_LAUNCH_CHECK("score_exact_fill");
    const int nsm = num_sms();
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
    {
        const int smem = (int)sizeof(XbSmem) + 128;
        if ((rc = ensure_smem_attr(reinterpret_cast<const void*>(score_exact_rowsum), smem))) return rc;
        score_exact_rowsum<<<(n_rows + XB_ROWS - 1) / XB_ROWS, XB_THREADS, smem, st>>>(
            mx, L, lq, n_rows, rowmax, rowsum);
        TSA_LAUNCH_CHECK("score_exact_rowsum");
    }
    {
        dim3 grid((L + XC_T - 1) / XC_T, nh);
        score_exact_colsum<<<grid, XC_T, sizeof(float) * 2 * lq, st>>>(X, L, Lp, lq, d.head_begin,
                                                                         rowmax, rowsum, colraw);
        TSA_LAUNCH_CHECK("score_exact_colsum");
    }
    tsa_desc pd = d;
    pd.last_q = 1;
    return launch_colsum_pool(pd, colraw, s, st);
}

}  // namespace tsa
