// Producer / consumer of the attention branch (layer_forward, model.cpp:169-201):
// the kernels around the path that cfg4's 32-layer prefill stack needs.
//
//   rms_norm          model.cpp:81-94   one thread per row sums x^2 sequentially
//                                       (f32, j ascending, FMUL then FADD -- the
//                                       reference's order, so f32 inputs match it
//                                       bit for bit); a warp per row scales
//   rope table        model.cpp:107-116 angle = pos * theta^(-2i/d) in double (the
//                                       frequencies come from the host's pow, as in
//                                       the reference), cos/sin in double -> f32
//   split_heads_rope  model.cpp:128-158 projection rows [L, (H + 2 Hkv) d] -> q
//                                       [H, L, d], k / v [Hkv, L, d], RoPE on q and
//                                       k in f32 (x0 c - x1 s, x0 s + x1 c, no FMA)
//   heads_concat      model.cpp:196-200 [H, L, d] -> [L, H d] for the W_O GEMM
//   layer_drift       drift.cpp:14-45   per token |h'[t] - h[t]| / (|h[t]| + eps)
//                                       with the sums in double, j ascending, then
//                                       the token mean summed t ascending (the
//                                       reference's order: bit-exact for f32)
//
// These are the unfused stages (a caller's BLAS does the projections between
// them); the cfg4 stack runs the fused tcgen05 projections of proj_gemm.cu
// instead.  Everything here is HBM-bound byte movement.
#include <cmath>

#include "common.cuh"

namespace tsa {
namespace {

template <typename T>
__device__ __forceinline__ float ld_f32(const T* p) {
    return Elem<T>::to_f32(*p);
}

// A CTA owns 32 rows.  Pass 1 streams the rows through shared memory in
// 128-column chunks (all 256 threads load, coalesced, double-buffered) while
// warp 0 -- one lane per row -- accumulates x^2 sequentially in the
// reference's order; pass 2 scales the rows with coalesced 16-byte accesses:
// out = (x * inv) * gain.
constexpr int RMS_ROWS = 32;
constexpr int RMS_CHUNK = 128;
constexpr int RMS_THREADS = 256;

template <typename T>
__global__ void __launch_bounds__(RMS_THREADS) rms_norm_kernel(const T* __restrict__ x,
                                                              const float* __restrict__ gain,
                                                              int64_t rows, int cols, float eps,
                                                              T* __restrict__ out) {
    __shared__ float chunk[2][RMS_ROWS][RMS_CHUNK + 1];  // +1: conflict-free row walks
    __shared__ float inv_s[RMS_ROWS];
    const int64_t r0 = (int64_t)blockIdx.x * RMS_ROWS;
    const int nrows = rows - r0 < RMS_ROWS ? (int)(rows - r0) : RMS_ROWS;
    const int tid = threadIdx.x;
    const int n_chunks = (cols + RMS_CHUNK - 1) / RMS_CHUNK;
    auto load = [&](int c, int buf) {
        const int c0 = c * RMS_CHUNK;
        for (int e = tid; e < RMS_ROWS * RMS_CHUNK; e += RMS_THREADS) {
            const int rr = e / RMS_CHUNK, j = e % RMS_CHUNK;
            float v = 0.0f;
            if (rr < nrows && c0 + j < cols) v = ld_f32(x + (r0 + rr) * cols + c0 + j);
            chunk[buf][rr][j] = v;
        }
    };
    float ss = 0.0f;
    load(0, 0);
    __syncthreads();
    for (int c = 0; c < n_chunks; ++c) {
        if (c + 1 < n_chunks) load(c + 1, (c + 1) & 1);  // overlaps warp 0's sums
        if (tid < RMS_ROWS) {
            const float* row = chunk[c & 1][tid];
            const int n = min(RMS_CHUNK, cols - c * RMS_CHUNK);
            for (int j = 0; j < n; ++j) ss = __fadd_rn(ss, __fmul_rn(row[j], row[j]));
        }
        __syncthreads();
    }
    // inv = 1 / sqrt(ss / cols + eps) (model.cpp:89), each step correctly rounded
    if (tid < RMS_ROWS)
        inv_s[tid] = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(__fdiv_rn(ss, (float)cols), eps)));
    __syncthreads();
    for (int rr = tid >> 5; rr < nrows; rr += RMS_THREADS / 32) {
        const float iv = inv_s[rr];
        const T* xr = x + (r0 + rr) * cols;
        T* o = out + (r0 + rr) * cols;
        for (int j = tid & 31; j < cols; j += 32)
            o[j] = Elem<T>::from_f32(__fmul_rn(__fmul_rn(ld_f32(xr + j), iv), gain[j]));
    }
}

struct RopeFreqs {
    double f[128];  // theta^(-2i/d), i < d/2 <= 128
};

__global__ void rope_table_kernel(const __grid_constant__ RopeFreqs freq, int seq_len, int half,
                                  float2* __restrict__ table) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (int64_t)seq_len * half) return;
    const int t = (int)(e / half), i = (int)(e % half);
    const double angle = (double)t * freq.f[i];
    double s, c;
    sincos(angle, &s, &c);
    table[e] = make_float2((float)c, (float)s);
}

// One thread per (row, head slot, group of 4 pairs).  Slots [0, H) are q
// heads, [H, H+Hkv) k heads, [H+Hkv, H+2Hkv) v heads of the projection row.
constexpr int ROPE_PAIRS = 4;

template <typename T>
__global__ void __launch_bounds__(256) split_heads_rope_kernel(
    const T* __restrict__ qkv, const float2* __restrict__ table, int L, int H, int Hkv, int d,
    T* __restrict__ q, T* __restrict__ k, T* __restrict__ v) {
    const int half = d / 2, groups = half / ROPE_PAIRS, slots = H + 2 * Hkv;
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (int64_t)L * slots * groups) return;
    const int g = (int)(e % groups);
    const int slot = (int)((e / groups) % slots);
    const int t = (int)(e / ((int64_t)groups * slots));
    const int i0 = g * ROPE_PAIRS;
    const T* src = qkv + ((int64_t)t * slots + slot) * d + 2 * i0;
    // 8 elements: one 16-B load for bf16, two for f32
    float xv[2 * ROPE_PAIRS];
    if constexpr (sizeof(T) == 2) {
        const uint4 raw = *reinterpret_cast<const uint4*>(src);
        const __nv_bfloat162* p2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
        for (int u = 0; u < ROPE_PAIRS; ++u) {
            const float2 f = __bfloat1622float2(p2[u]);
            xv[2 * u] = f.x;
            xv[2 * u + 1] = f.y;
        }
    } else {
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const float4 f = reinterpret_cast<const float4*>(src)[u];
            xv[4 * u] = f.x;
            xv[4 * u + 1] = f.y;
            xv[4 * u + 2] = f.z;
            xv[4 * u + 3] = f.w;
        }
    }
    T* dst;
    if (slot < H + Hkv) {
        const float4* tb4 = reinterpret_cast<const float4*>(table + (int64_t)t * half + i0);
        const float4 cs01 = tb4[0], cs23 = tb4[1];
        const float2 tb[ROPE_PAIRS] = {make_float2(cs01.x, cs01.y), make_float2(cs01.z, cs01.w),
                                       make_float2(cs23.x, cs23.y), make_float2(cs23.z, cs23.w)};
#pragma unroll
        for (int u = 0; u < ROPE_PAIRS; ++u) {
            const float2 cs = tb[u];
            const float x0 = xv[2 * u], x1 = xv[2 * u + 1];
            xv[2 * u] = __fsub_rn(__fmul_rn(x0, cs.x), __fmul_rn(x1, cs.y));
            xv[2 * u + 1] = __fadd_rn(__fmul_rn(x0, cs.y), __fmul_rn(x1, cs.x));
        }
        dst = slot < H ? q + ((int64_t)slot * L + t) * d : k + ((int64_t)(slot - H) * L + t) * d;
    } else {
        dst = v + ((int64_t)(slot - H - Hkv) * L + t) * d;
    }
    if constexpr (sizeof(T) == 2) {
        uint4 raw;
        __nv_bfloat162* p2 = reinterpret_cast<__nv_bfloat162*>(&raw);
#pragma unroll
        for (int u = 0; u < ROPE_PAIRS; ++u) p2[u] = __floats2bfloat162_rn(xv[2 * u], xv[2 * u + 1]);
        *reinterpret_cast<uint4*>(dst + 2 * i0) = raw;
    } else {
#pragma unroll
        for (int u = 0; u < 2; ++u)
            reinterpret_cast<float4*>(dst + 2 * i0)[u] =
                make_float4(xv[4 * u], xv[4 * u + 1], xv[4 * u + 2], xv[4 * u + 3]);
    }
}

// cat[t, h d + c] = heads[h, t, c]; 16-byte units.
__global__ void __launch_bounds__(256) heads_concat_kernel(const uint4* __restrict__ heads, int L,
                                                          int H, int units_per_row,
                                                          uint4* __restrict__ cat) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t total = (int64_t)L * H * units_per_row;
    if (e >= total) return;
    const int c = (int)(e % units_per_row);
    const int h = (int)((e / units_per_row) % H);
    const int64_t t = e / ((int64_t)units_per_row * H);
    cat[e] = heads[((int64_t)h * L + t) * units_per_row + c];
}

// Drift of one layer boundary, pass 1: a CTA owns 32 tokens; both matrices
// stream through shared memory in 128-column chunks and lane t of warp 0
// accumulates num = sum (b - a)^2 and den = sum a^2 in double, j ascending.
constexpr int DR_ROWS = 32, DR_CHUNK = 128, DR_THREADS = 256;

template <typename T>
__global__ void __launch_bounds__(DR_THREADS) drift_ratio_kernel(const T* __restrict__ a,
                                                                const T* __restrict__ b,
                                                                int64_t rows, int cols,
                                                                double eps,
                                                                double* __restrict__ ratio) {
    __shared__ float ca[DR_ROWS][DR_CHUNK + 1], cb[DR_ROWS][DR_CHUNK + 1];
    const int64_t r0 = (int64_t)blockIdx.x * DR_ROWS;
    const int nrows = rows - r0 < DR_ROWS ? (int)(rows - r0) : DR_ROWS;
    const int tid = threadIdx.x;
    double num = 0.0, den = 0.0;
    for (int c0 = 0; c0 < cols; c0 += DR_CHUNK) {
        const int n = min(DR_CHUNK, cols - c0);
        for (int e = tid; e < DR_ROWS * DR_CHUNK; e += DR_THREADS) {
            const int rr = e / DR_CHUNK, j = e % DR_CHUNK;
            float va = 0.0f, vb = 0.0f;
            if (rr < nrows && j < n) {
                va = ld_f32(a + (r0 + rr) * cols + c0 + j);
                vb = ld_f32(b + (r0 + rr) * cols + c0 + j);
            }
            ca[rr][j] = va;
            cb[rr][j] = vb;
        }
        __syncthreads();
        if (tid < DR_ROWS) {
            for (int j = 0; j < n; ++j) {
                const double x = (double)ca[tid][j];
                const double d = __dsub_rn((double)cb[tid][j], x);
                num = __dadd_rn(num, __dmul_rn(d, d));
                den = __dadd_rn(den, __dmul_rn(x, x));
            }
        }
        __syncthreads();
    }
    if (tid < nrows)
        ratio[r0 + tid] = __ddiv_rn(__dsqrt_rn(num), __dadd_rn(__dsqrt_rn(den), eps));
}

// Pass 2: the token mean, summed sequentially (t ascending) as the reference does.
__global__ void drift_mean_kernel(const double* __restrict__ ratio, int64_t rows,
                                  double* __restrict__ out) {
    double acc = 0.0;
    for (int64_t t = 0; t < rows; ++t) acc = __dadd_rn(acc, ratio[t]);
    *out = __ddiv_rn(acc, (double)rows);
}

}  // namespace

int launch_rms_norm(const void* x, const float* gain, int64_t rows, int cols, float eps, int dtype,
                    void* out, cudaStream_t st) {
    const unsigned grid = (unsigned)((rows + RMS_ROWS - 1) / RMS_ROWS);
    if (dtype == TSA_BF16)
        rms_norm_kernel<__nv_bfloat16><<<grid, RMS_THREADS, 0, st>>>(
            (const __nv_bfloat16*)x, gain, rows, cols, eps, (__nv_bfloat16*)out);
    else
        rms_norm_kernel<float><<<grid, RMS_THREADS, 0, st>>>((const float*)x, gain, rows, cols,
                                                             eps, (float*)out);
    TSA_LAUNCH_CHECK("rms_norm");
    return 0;
}

int launch_rope_table(int seq_len, int d_head, float theta, float* table, cudaStream_t st) {
    const int half = d_head / 2;
    if (half < 1 || half > 128) return invalid("rope_table: d_head must be in [2, 256]");
    // theta^(-2i/d) in double on the host: the reference's own expression and libm
    RopeFreqs f{};
    for (int i = 0; i < half; ++i)
        f.f[i] = std::pow(static_cast<double>(theta), -2.0 * static_cast<double>(i) /
                                                          static_cast<double>(d_head));
    const int64_t n = (int64_t)seq_len * half;
    rope_table_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(f, seq_len, half,
                                                                  reinterpret_cast<float2*>(table));
    TSA_LAUNCH_CHECK("rope_table");
    return 0;
}

int launch_split_heads_rope(const tsa_desc& d, const void* qkv, const float* table, void* q,
                            void* k, void* v, cudaStream_t st) {
    const int L = d.seq_len, H = d.n_heads, Hkv = d.n_kv_heads, D = d.d_head;
    if ((D / 2) % ROPE_PAIRS != 0)
        return invalid("split_heads_rope: d_head must be a multiple of " +
                       std::to_string(2 * ROPE_PAIRS));
    const int64_t n = (int64_t)L * (H + 2 * Hkv) * (D / 2 / ROPE_PAIRS);
    const unsigned grid = (unsigned)((n + 255) / 256);
    const float2* tb = reinterpret_cast<const float2*>(table);
    if (d.dtype == TSA_BF16)
        split_heads_rope_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(
            (const __nv_bfloat16*)qkv, tb, L, H, Hkv, D, (__nv_bfloat16*)q, (__nv_bfloat16*)k,
            (__nv_bfloat16*)v);
    else
        split_heads_rope_kernel<float><<<grid, 256, 0, st>>>((const float*)qkv, tb, L, H, Hkv, D,
                                                             (float*)q, (float*)k, (float*)v);
    TSA_LAUNCH_CHECK("split_heads_rope");
    return 0;
}

int launch_heads_concat(const tsa_desc& d, const void* heads, void* cat, cudaStream_t st) {
    const size_t row_bytes = (size_t)d.d_head * elem_bytes(d.dtype);
    if (row_bytes % 16) return invalid("heads_concat: head rows must be a multiple of 16 bytes");
    const int upr = (int)(row_bytes / 16);
    const int64_t n = (int64_t)d.seq_len * d.n_heads * upr;
    heads_concat_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
        (const uint4*)heads, d.seq_len, d.n_heads, upr, (uint4*)cat);
    TSA_LAUNCH_CHECK("heads_concat");
    return 0;
}

}  // namespace tsa

namespace tsa {

int launch_layer_drift(const void* prev, const void* next, int64_t rows, int cols, int dtype,
                       double eps, double* out, double* ratio_ws, cudaStream_t st) {
    const unsigned grid = (unsigned)((rows + DR_ROWS - 1) / DR_ROWS);
    if (dtype == TSA_BF16)
        drift_ratio_kernel<__nv_bfloat16><<<grid, DR_THREADS, 0, st>>>(
            (const __nv_bfloat16*)prev, (const __nv_bfloat16*)next, rows, cols, eps, ratio_ws);
    else
        drift_ratio_kernel<float><<<grid, DR_THREADS, 0, st>>>((const float*)prev,
                                                               (const float*)next, rows, cols,
                                                               eps, ratio_ws);
    TSA_LAUNCH_CHECK("drift_ratio");
    drift_mean_kernel<<<1, 1, 0, st>>>(ratio_ws, rows, out);
    TSA_LAUNCH_CHECK("drift_mean");
    return 0;
}

}  // namespace tsa
