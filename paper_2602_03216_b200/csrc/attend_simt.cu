// K5 (SIMT variant): causal flash attention in f32 arithmetic for any
// supported head size, used for the f32 configuration (parity gate 1e-5,
// bench.cpp:27) and for bf16 shapes the tcgen05 kernel does not cover.
//
// dense_causal_attention (attention.cpp:25-40) over the first n rows of each
// head: O[i] = sum_{j<=i} softmax_j(q_i . k_j / sqrt(d)) v_j, computed with
// the online (tile-wise) softmax.  n comes from device memory (k_keep), so
// the grid is sized for L and surplus tiles exit immediately.
//
// Block = 32 query rows x 4 threads per row; a thread owns the 16-B chunks
// c = part, part+4, ... of its row (conflict-free shared-memory reads).
#include <cstdlib>

#include "common.cuh"

namespace tsa {
namespace {

constexpr int SM_ROWS = 32;
constexpr int SM_KEYS = 32;

template <typename T, int D>
__global__ void __launch_bounds__(128) attend_simt_kernel(const T* __restrict__ q,
                                                          const T* __restrict__ k,
                                                          const T* __restrict__ v,
                                                          const int32_t* __restrict__ n_dev,
                                                          int n_const, int kv_group,
                                                          int rows_per_head, int kv_rows_per_head,
                                                          int head_begin, float scale,
                                                          T* __restrict__ o) {
    constexpr int NC = D / 4;        // float4 chunks per row
    constexpr int CPT = NC / 4 > 0 ? NC / 4 : 1;  // chunks per thread
    extern __shared__ float4 smem4[];
    float4* ks = smem4;                // [SM_KEYS][NC]
    float4* vs = smem4 + SM_KEYS * NC; // [SM_KEYS][NC]

    const int h = head_begin + blockIdx.y;
    const int n = n_dev ? *n_dev : n_const;
    const int n_tiles = (n + SM_ROWS - 1) / SM_ROWS;
    if ((int)blockIdx.x >= n_tiles) return;
    const int tile = n_tiles - 1 - blockIdx.x;  // heaviest (longest causal row) first
    const int row_in = threadIdx.x / 4, part = threadIdx.x % 4;
    const int i = tile * SM_ROWS + row_in;
    const bool active_part = part < NC;  // D = 8: only 2 chunks per row
    const int kvh = h / kv_group;
    const T* qh = q + (size_t)h * rows_per_head * D;
    const T* kh = k + (size_t)kvh * kv_rows_per_head * D;
    const T* vh = v + (size_t)kvh * kv_rows_per_head * D;

    float4 qr[CPT], acc[CPT];
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
        acc[c] = make_float4(0.f, 0.f, 0.f, 0.f);
        qr[c] = make_float4(0.f, 0.f, 0.f, 0.f);
        const int ch = part + 4 * c;
        if (i < n && active_part && ch < NC) {
            const T* src = qh + (size_t)i * D + ch * 4;
            qr[c] = make_float4(Elem<T>::to_f32(src[0]), Elem<T>::to_f32(src[1]),
                                Elem<T>::to_f32(src[2]), Elem<T>::to_f32(src[3]));
        }
    }
    float m = -INFINITY, l = 0.0f;
    const int last_key = min(n, (tile + 1) * SM_ROWS) - 1;
    for (int j0 = 0; j0 <= last_key; j0 += SM_KEYS) {
        __syncthreads();
        for (int e = threadIdx.x; e < SM_KEYS * NC; e += 128) {
            const int j = e / NC, ch = e % NC;
            float4 kk = make_float4(0.f, 0.f, 0.f, 0.f), vv = kk;
            if (j0 + j <= last_key) {
                const T* ksrc = kh + (size_t)(j0 + j) * D + ch * 4;
                const T* vsrc = vh + (size_t)(j0 + j) * D + ch * 4;
                kk = make_float4(Elem<T>::to_f32(ksrc[0]), Elem<T>::to_f32(ksrc[1]),
                                 Elem<T>::to_f32(ksrc[2]), Elem<T>::to_f32(ksrc[3]));
                vv = make_float4(Elem<T>::to_f32(vsrc[0]), Elem<T>::to_f32(vsrc[1]),
                                 Elem<T>::to_f32(vsrc[2]), Elem<T>::to_f32(vsrc[3]));
            }
            ks[j * NC + ch] = kk;
            vs[j * NC + ch] = vv;
        }
        __syncthreads();
        float sc[SM_KEYS];
        float tmax = -INFINITY;
#pragma unroll
        for (int j = 0; j < SM_KEYS; ++j) {
            float p = 0.f;
#pragma unroll
            for (int c = 0; c < CPT; ++c) {
                const int ch = part + 4 * c;
                if (active_part && ch < NC) {
                    const float4 kk = ks[j * NC + ch];
                    p = fmaf(qr[c].x, kk.x, p);
                    p = fmaf(qr[c].y, kk.y, p);
                    p = fmaf(qr[c].z, kk.z, p);
                    p = fmaf(qr[c].w, kk.w, p);
                }
            }
            p += __shfl_xor_sync(0xffffffffu, p, 1);
            p += __shfl_xor_sync(0xffffffffu, p, 2);
            const int jj = j0 + j;
            sc[j] = (jj <= i && jj <= last_key) ? p * scale : -INFINITY;
            tmax = fmaxf(tmax, sc[j]);
        }
        const float m_new = fmaxf(m, tmax);
        if (m_new == -INFINITY) continue;  // rows beyond n: nothing allowed yet
        const float corr = expf(m - m_new);
        l *= corr;
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
            acc[c].x *= corr;
            acc[c].y *= corr;
            acc[c].z *= corr;
            acc[c].w *= corr;
        }
#pragma unroll
        for (int j = 0; j < SM_KEYS; ++j) {
            const float p = expf(sc[j] - m_new);
            l += p;
#pragma unroll
            for (int c = 0; c < CPT; ++c) {
                const int ch = part + 4 * c;
                if (active_part && ch < NC) {
                    const float4 vv = vs[j * NC + ch];
                    acc[c].x = fmaf(p, vv.x, acc[c].x);
                    acc[c].y = fmaf(p, vv.y, acc[c].y);
                    acc[c].z = fmaf(p, vv.z, acc[c].z);
                    acc[c].w = fmaf(p, vv.w, acc[c].w);
                }
            }
        }
        m = m_new;
    }
    if (i >= n) return;
    const float inv_l = 1.0f / l;
    T* dst = o + ((size_t)h * rows_per_head + i) * D;
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
        const int ch = part + 4 * c;
        if (active_part && ch < NC) {
            dst[ch * 4 + 0] = Elem<T>::from_f32(acc[c].x * inv_l);
            dst[ch * 4 + 1] = Elem<T>::from_f32(acc[c].y * inv_l);
            dst[ch * 4 + 2] = Elem<T>::from_f32(acc[c].z * inv_l);
            dst[ch * 4 + 3] = Elem<T>::from_f32(acc[c].w * inv_l);
        }
    }
}

// f32 inputs, d = 128 (cfg1): register-tiled flash attention on the CUDA
// cores.  Block = 64 query rows x 32-key tiles, 128 threads; thread t owns
// rows 4*(t/8) .. +3 and, for S = Q K^T, keys 4*(t%8) .. +3 (a 4 x 4 tile:
// one float4 of Q and one of K per dim feed 16 FMAs), for O += P V the float4
// column chunks (t%8) + 8c, c < 4 (64 accumulators; the 8 threads of a row
// group read 128 contiguous bytes of V -- conflict-free).  Q and K sit in
// shared memory transposed ([d][row], [d][key]) so those reads are single
// float4s; P goes through shared memory transposed ([key][row]).  Row max /
// sum over a key tile: shuffles among the 8 threads of the row group.  Exact
// f32 online softmax (expf), fma accumulation: within the reference's 1e-5
// gate (bench.cpp:27) of its non-fused order.
constexpr int TR = 64, TK = 32, TD = 128;

template <typename T>
__global__ void __launch_bounds__(128) attend_tiled_d128(const T* __restrict__ q,
                                                         const T* __restrict__ k,
                                                         const T* __restrict__ v,
                                                         const int32_t* __restrict__ n_dev,
                                                         int n_const, int kv_group,
                                                         int rows_per_head, int kv_rows_per_head,
                                                         int head_begin, float scale,
                                                         T* __restrict__ o) {
    static_assert(sizeof(T) == 4, "cp.async K/V staging copies f32 elements");
    extern __shared__ float4 smem4[];
    float* Qs = reinterpret_cast<float*>(smem4);  // [TD][TR]
    float* Kb = Qs + TD * TR;                     // 2 x [TD][TK]
    float* Vb = Kb + 2 * TD * TK;                 // 2 x [TK][TD]
    float* Ps = Vb + 2 * TK * TD;                 // [TK][TR]
    const int tid = threadIdx.x;
    const int h = head_begin + blockIdx.y;
    const int n = n_dev ? *n_dev : n_const;
    const int n_tiles = (n + TR - 1) / TR;
    if ((int)blockIdx.x >= n_tiles) return;
    const int r0 = (n_tiles - 1 - (int)blockIdx.x) * TR;  // heaviest first
    const int kvh = h / kv_group;
    const T* qh = q + (size_t)h * rows_per_head * TD;
    const T* kh = k + (size_t)kvh * kv_rows_per_head * TD;
    const T* vh = v + (size_t)kvh * kv_rows_per_head * TD;
    const int rg = tid >> 3, cg = tid & 7;  // row group (4 rows), key / column group

    // Q tile, transposed: thread -> (row = e % 64, dim chunk = e / 64)
    for (int e = tid; e < TR * (TD / 4); e += 128) {
        const int r = e % TR, c4 = e / TR;
        float x[4] = {0.f, 0.f, 0.f, 0.f};
        if (r0 + r < n) {
            const T* src = qh + (size_t)(r0 + r) * TD + c4 * 4;
#pragma unroll
            for (int u = 0; u < 4; ++u) x[u] = Elem<T>::to_f32(src[u]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) Qs[(c4 * 4 + u) * TR + r] = x[u];
    }
    float acc[4][16];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 16; ++c) acc[r][c] = 0.f;
    float m[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY}, l[4] = {0.f, 0.f, 0.f, 0.f};
    const int last_key = min(n, r0 + TR) - 1;
    // K (transposed, 4-byte copies) and V (16-byte copies) of key tile j0 into
    // buffer b with cp.async, zero-filled past last_key: the next tile's loads
    // are in flight while the current one computes
    auto prefetch = [&](int j0, int b) {
        float* Ks = Kb + b * TD * TK;
        float* Vs = Vb + b * TK * TD;
        for (int e = tid; e < TK * TD; e += 128) {
            const int key = e % TK, dd = e / TK;  // a warp covers 32 keys of one dim
            const bool ok = j0 + key <= last_key;
            const T* src = kh + (size_t)(ok ? j0 + key : 0) * TD + dd;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(
                             (uint32_t)__cvta_generic_to_shared(Ks + dd * TK + key)),
                         "l"(src), "r"(ok ? 4 : 0));
        }
        for (int e = tid; e < TK * (TD / 4); e += 128) {
            const int key = e / (TD / 4), c4 = e % (TD / 4);
            const bool ok = j0 + key <= last_key;
            const T* src = vh + (size_t)(ok ? j0 + key : 0) * TD + c4 * 4;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(
                             (uint32_t)__cvta_generic_to_shared(Vs + key * TD + c4 * 4)),
                         "l"(src), "r"(ok ? 16 : 0));
        }
        asm volatile("cp.async.commit_group;\n" ::);
    };
    prefetch(0, 0);
    for (int j0 = 0, b = 0; j0 <= last_key; j0 += TK, b ^= 1) {
        asm volatile("cp.async.wait_group 0;\n" ::);
        __syncthreads();  // tile j0 landed for every thread; tile j0 - TK fully consumed
        if (j0 + TK <= last_key) prefetch(j0 + TK, b ^ 1);
        const float* Ks = Kb + b * TD * TK;
        const float* Vs = Vb + b * TK * TD;
        // S tile 4 x 4
        float sc[4][4];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c) sc[r][c] = 0.f;
#pragma unroll 8
        for (int d = 0; d < TD; ++d) {
            const float4 qa = reinterpret_cast<const float4*>(Qs + d * TR)[rg];
            const float4 kb = reinterpret_cast<const float4*>(Ks + d * TK)[cg];
            const float qv[4] = {qa.x, qa.y, qa.z, qa.w}, kv[4] = {kb.x, kb.y, kb.z, kb.w};
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int c = 0; c < 4; ++c) sc[r][c] = fmaf(qv[r], kv[c], sc[r][c]);
        }
        float corr[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int i = r0 + rg * 4 + r;
            float tmax = -INFINITY;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const int key = j0 + cg * 4 + c;
                sc[r][c] = (key <= i && key <= last_key) ? sc[r][c] * scale : -INFINITY;
                tmax = fmaxf(tmax, sc[r][c]);
            }
            tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 1));
            tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 2));
            tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 4));
            const float m_new = fmaxf(m[r], tmax);
            float psum = 0.f;
            if (m_new == -INFINITY) {  // no key visible yet (rows >= n)
                corr[r] = 1.f;
#pragma unroll
                for (int c = 0; c < 4; ++c) sc[r][c] = 0.f;
            } else {
                corr[r] = expf(m[r] - m_new);
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    sc[r][c] = expf(sc[r][c] - m_new);
                    psum += sc[r][c];
                }
            }
            psum += __shfl_xor_sync(0xffffffffu, psum, 1);
            psum += __shfl_xor_sync(0xffffffffu, psum, 2);
            psum += __shfl_xor_sync(0xffffffffu, psum, 4);
            l[r] = l[r] * corr[r] + psum;
            m[r] = m_new;
        }
#pragma unroll
        for (int c = 0; c < 4; ++c)
            reinterpret_cast<float4*>(Ps + (cg * 4 + c) * TR)[rg] =
                make_float4(sc[0][c], sc[1][c], sc[2][c], sc[3][c]);
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int c = 0; c < 16; ++c) acc[r][c] *= corr[r];
        __syncthreads();
        // O += P V over the tile's keys
#pragma unroll 4
        for (int j = 0; j < TK; ++j) {
            const float4 pa = reinterpret_cast<const float4*>(Ps + j * TR)[rg];
            const float pv[4] = {pa.x, pa.y, pa.z, pa.w};
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const float4 vb = reinterpret_cast<const float4*>(Vs + j * TD)[cg + 8 * c];
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    acc[r][c * 4 + 0] = fmaf(pv[r], vb.x, acc[r][c * 4 + 0]);
                    acc[r][c * 4 + 1] = fmaf(pv[r], vb.y, acc[r][c * 4 + 1]);
                    acc[r][c * 4 + 2] = fmaf(pv[r], vb.z, acc[r][c * 4 + 2]);
                    acc[r][c * 4 + 3] = fmaf(pv[r], vb.w, acc[r][c * 4 + 3]);
                }
            }
        }
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int i = r0 + rg * 4 + r;
        if (i >= n) continue;
        const float inv_l = 1.0f / l[r];
        T* dst = o + ((size_t)h * rows_per_head + i) * TD;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int col = (cg + 8 * c) * 4;
            dst[col + 0] = Elem<T>::from_f32(acc[r][c * 4 + 0] * inv_l);
            dst[col + 1] = Elem<T>::from_f32(acc[r][c * 4 + 1] * inv_l);
            dst[col + 2] = Elem<T>::from_f32(acc[r][c * 4 + 2] * inv_l);
            dst[col + 3] = Elem<T>::from_f32(acc[r][c * 4 + 3] * inv_l);
        }
    }
}

int launch_tiled_d128_f32(const tsa_desc& d, const void* q, const void* k, const void* v,
                          const int32_t* n_dev, int n_const, int kv_group, int rph, int kvrph,
                          void* o, cudaStream_t st) {
    const int nh = d.head_end - d.head_begin;
    dim3 grid((d.seq_len + TR - 1) / TR, nh);
    const int smem = (TD * TR + 2 * TD * TK + 2 * TK * TD + TK * TR) * (int)sizeof(float);
    if (int rc = ensure_smem_attr(reinterpret_cast<const void*>(attend_tiled_d128<float>), smem))
        return rc;
    attend_tiled_d128<float><<<grid, 128, smem, st>>>((const float*)q, (const float*)k,
                                                      (const float*)v, n_dev, n_const, kv_group,
                                                      rph, kvrph, d.head_begin,
                                                      1.0f / sqrtf((float)TD), (float*)o);
    TSA_LAUNCH_CHECK("attend_tiled_d128");
    return 0;
}

// Any other head size (the reference's unit tests use d = 1 and 4): one
// thread per query row, per-key online softmax, K/V straight from global.
template <typename T>
__global__ void __launch_bounds__(128) attend_simt_any_d(const T* __restrict__ q,
                                                         const T* __restrict__ k,
                                                         const T* __restrict__ v,
                                                         const int32_t* __restrict__ n_dev,
                                                         int n_const, int kv_group,
                                                         int rows_per_head, int kv_rows_per_head,
                                                         int head_begin, int D, float scale,
                                                         T* __restrict__ o) {
    constexpr int DMAX = 256;
    const int h = head_begin + blockIdx.y;
    const int n = n_dev ? *n_dev : n_const;
    const int i = blockIdx.x * 128 + threadIdx.x;
    if (i >= n) return;
    const int kvh = h / kv_group;
    const T* qi = q + ((size_t)h * rows_per_head + i) * D;
    const T* kh = k + (size_t)kvh * kv_rows_per_head * D;
    const T* vh = v + (size_t)kvh * kv_rows_per_head * D;
    float qr[DMAX], acc[DMAX];
    for (int p = 0; p < D; ++p) {
        qr[p] = Elem<T>::to_f32(qi[p]);
        acc[p] = 0.0f;
    }
    float m = -INFINITY, l = 0.0f;
    for (int j = 0; j <= i; ++j) {
        float s = 0.0f;
        for (int p = 0; p < D; ++p) s = fmaf(qr[p], Elem<T>::to_f32(kh[(size_t)j * D + p]), s);
        s *= scale;
        const float m_new = fmaxf(m, s);
        const float corr = expf(m - m_new);
        const float pj = expf(s - m_new);
        l = l * corr + pj;
        for (int p = 0; p < D; ++p)
            acc[p] = fmaf(pj, Elem<T>::to_f32(vh[(size_t)j * D + p]), acc[p] * corr);
        m = m_new;
    }
    T* dst = o + ((size_t)h * rows_per_head + i) * D;
    const float inv_l = 1.0f / l;
    for (int p = 0; p < D; ++p) dst[p] = Elem<T>::from_f32(acc[p] * inv_l);
}

template <typename T, int D>
int launch_t(const tsa_desc& d, const void* q, const void* k, const void* v, const int32_t* n_dev,
             int n_const, int kv_group, int rows_per_head, int kv_rows_per_head, void* o,
             cudaStream_t st) {
    const int nh = d.head_end - d.head_begin;
    dim3 grid((d.seq_len + SM_ROWS - 1) / SM_ROWS, nh);
    const size_t smem = 2 * SM_KEYS * (D / 4) * sizeof(float4);
    auto kern = attend_simt_kernel<T, D>;
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<grid, 128, smem, st>>>((const T*)q, (const T*)k, (const T*)v, n_dev, n_const, kv_group,
                                  rows_per_head, kv_rows_per_head, d.head_begin,
                                  1.0f / sqrtf((float)D), (T*)o);
    TSA_LAUNCH_CHECK("attend_simt");
    return 0;
}

template <typename T>
int dispatch_d(const tsa_desc& d, const void* q, const void* k, const void* v,
               const int32_t* n_dev, int n_const, int kv_group, int rph, int kvrph, void* o,
               cudaStream_t st) {
    switch (d.d_head) {
        case 8: return launch_t<T, 8>(d, q, k, v, n_dev, n_const, kv_group, rph, kvrph, o, st);
        case 16: return launch_t<T, 16>(d, q, k, v, n_dev, n_const, kv_group, rph, kvrph, o, st);
        case 32: return launch_t<T, 32>(d, q, k, v, n_dev, n_const, kv_group, rph, kvrph, o, st);
        case 64: return launch_t<T, 64>(d, q, k, v, n_dev, n_const, kv_group, rph, kvrph, o, st);
        case 128:
            if (sizeof(T) == 4 && !std::getenv("TSA_SIMT_ROWWISE"))  // f32: register-tiled
                return launch_tiled_d128_f32(d, q, k, v, n_dev, n_const, kv_group, rph, kvrph,
                                             o, st);
            return launch_t<T, 128>(d, q, k, v, n_dev, n_const, kv_group, rph, kvrph, o, st);
        case 256: return launch_t<T, 256>(d, q, k, v, n_dev, n_const, kv_group, rph, kvrph, o, st);
        default: {
            if (d.d_head < 1 || d.d_head > 256)
                return invalid("attend: unsupported d_head " + std::to_string(d.d_head));
            dim3 grid((d.seq_len + 127) / 128, d.head_end - d.head_begin);
            attend_simt_any_d<T><<<grid, 128, 0, st>>>(
                (const T*)q, (const T*)k, (const T*)v, n_dev, n_const, kv_group, rph, kvrph,
                d.head_begin, d.d_head, 1.0f / sqrtf((float)d.d_head), (T*)o);
            TSA_LAUNCH_CHECK("attend_simt_any_d");
            return 0;
        }
    }
}

}  // namespace

int launch_attend_simt(const tsa_desc& d, const void* q, const void* k, const void* v,
                       const int32_t* n_dev, int32_t n_const, int32_t kv_group,
                       int32_t rows_per_head, int32_t kv_rows_per_head, void* o, cudaStream_t st) {
    if (d.dtype == TSA_BF16)
        return dispatch_d<__nv_bfloat16>(d, q, k, v, n_dev, n_const, kv_group, rows_per_head,
                                         kv_rows_per_head, o, st);
    return dispatch_d<float>(d, q, k, v, n_dev, n_const, kv_group, rows_per_head,
                             kv_rows_per_head, o, st);
}

}  // namespace tsa
