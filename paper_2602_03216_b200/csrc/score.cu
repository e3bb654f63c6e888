// K1: per-head token-importance scoring (score_tokens, token_coverage.cpp:16-50).
//
// REFERENCE mode reproduces the reference's f32 arithmetic on the GPU:
//   logits  x[r, j] = (sum_p q[L-lq+r, p] * k[j, p]) * (1/sqrt(d))   p ascending, no FMA
//                                                                     (tensor_ops.cpp:19-23)
//   softmax e = exp(x - max) rounded to f32, sequential f32 row sum, divide
//                                                                     (tensor_ops.cpp:47-69)
//   colsum  c[j] = sum_r P[r, j]                                      r ascending (:43-46)
//   pool    edge-clamped mean with Eigen's SSE2 segment-sum order     (tensor_ops.cpp:114-129)
// so scores match the reference bit for bit (expf is glibc's algorithm ported
// exactly, expf_glibc.cuh).  This is the general path (f32 inputs, any d);
// bf16 with d = 128 runs the fused kernels of score_exact.cu.  Three launches:
//   score_logits_ref  -> logits[h, r, j] (only the causally allowed prefix)
//   score_softmax_ref -> in place: P[h, r, j]
//   score_colsum_ref  -> s[h, t] (column sums + pooling, halo of kernel/2)
#include <climits>

#include "common.cuh"
#include "chain_sum.cuh"
#include "expf_glibc.cuh"

namespace tsa {
namespace {

constexpr int LG_ROWS = 64;   // max lq rows handled per block (lq <= 64 per tile; more tiles if larger)
constexpr int LG_KEYS = 128;  // keys per block
constexpr int LG_PCH = 32;    // d-chunk staged in smem

// Four consecutive elements of a row as f32 (16-B / 8-B vector load).
__device__ __forceinline__ void load4(const float* p, float (&x)[4]) {
    const float4 v = *reinterpret_cast<const float4*>(p);
    x[0] = v.x, x[1] = v.y, x[2] = v.z, x[3] = v.w;
}
__device__ __forceinline__ void load4(const __nv_bfloat16* p, float (&x)[4]) {
    const uint2 v = *reinterpret_cast<const uint2*>(p);
    x[0] = __uint_as_float(v.x << 16), x[1] = __uint_as_float(v.x & 0xFFFF0000u);
    x[2] = __uint_as_float(v.y << 16), x[3] = __uint_as_float(v.y & 0xFFFF0000u);
}

// Block: 256 threads = 16 row-groups (4 rows) x 16 key-groups (8 keys: 4 at
// tk*4 and 4 at 64 + tk*4, so a half-warp's float4 reads of a staged key row
// are 256 contiguous bytes -- two wavefronts, no bank conflicts).  Each
// (row, key) dot product runs in p order with separate multiply and add
// (matmul in p order, tensor_ops.cpp:19-23, called at token_coverage.cpp:31).
template <typename T>
// Lp > 0: the exact scorer's layout -- rows (local head, r) at stride Lp, and
// each row's maximum (atomicMax of the ordered encoding into rowmax) for the
// exact row / column passes; Lp == 0: rows (head, r) at stride L.
__global__ void __launch_bounds__(256) score_logits_ref(const T* __restrict__ q, const T* __restrict__ k,
                                                        float* __restrict__ logits, int H, int group,
                                                        int L, int d, int lq, int head_begin,
                                                        float inv_sqrt_d, int Lp,
                                                        int* __restrict__ rowmax) {
    // pitches of 4 floats over the tile widths: rows stay 16-B aligned for the
    // float4 reads
    __shared__ __align__(16) float qs[LG_PCH][LG_ROWS + 4];
    __shared__ __align__(16) float ks[LG_PCH][LG_KEYS + 4];
    const int h = head_begin + blockIdx.y;
    const int r_base = blockIdx.z * LG_ROWS;
    const int j0 = blockIdx.x * LG_KEYS;
    // keys beyond the causal limit of the last row are never needed
    if (j0 > L - lq + min(lq - 1, r_base + LG_ROWS - 1)) return;
    const int kv = h / group;
    const T* qh = q + ((size_t)h * L + (L - lq)) * d;
    const T* kh = k + (size_t)kv * L * d;
    const int tr = threadIdx.x / 16, tk = threadIdx.x % 16;
    const bool vec = (d % LG_PCH) == 0;  // whole chunks: 4-element vector staging
    float acc[4][8];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 8; ++b) acc[a][b] = 0.0f;

    for (int p0 = 0; p0 < d; p0 += LG_PCH) {
        const int pn = min(LG_PCH, d - p0);
        __syncthreads();
        if (vec) {
            for (int e = threadIdx.x; e < LG_ROWS * LG_PCH / 4; e += 256) {
                const int r = e / (LG_PCH / 4), p4 = 4 * (e % (LG_PCH / 4));
                const int rr = r_base + r;
                float x[4] = {0.0f, 0.0f, 0.0f, 0.0f};
                if (rr < lq) load4(qh + (size_t)rr * d + p0 + p4, x);
#pragma unroll
                for (int i = 0; i < 4; ++i) qs[p4 + i][r] = x[i];
            }
            for (int e = threadIdx.x; e < LG_KEYS * LG_PCH / 4; e += 256) {
                const int j = e / (LG_PCH / 4), p4 = 4 * (e % (LG_PCH / 4));
                const int jj = j0 + j;
                float x[4] = {0.0f, 0.0f, 0.0f, 0.0f};
                if (jj < L) load4(kh + (size_t)jj * d + p0 + p4, x);
#pragma unroll
                for (int i = 0; i < 4; ++i) ks[p4 + i][j] = x[i];
            }
        } else {
            for (int e = threadIdx.x; e < LG_ROWS * LG_PCH; e += 256) {
                const int r = e / LG_PCH, p = e % LG_PCH;
                const int rr = r_base + r;
                qs[p][r] = (rr < lq && p < pn) ? Elem<T>::to_f32(qh[(size_t)rr * d + p0 + p]) : 0.0f;
            }
            for (int e = threadIdx.x; e < LG_KEYS * LG_PCH; e += 256) {
                const int j = e / LG_PCH, p = e % LG_PCH;
                const int jj = j0 + j;
                ks[p][j] = (jj < L && p < pn) ? Elem<T>::to_f32(kh[(size_t)jj * d + p0 + p]) : 0.0f;
            }
        }
        __syncthreads();
        for (int p = 0; p < pn; ++p) {
            const float4 qv = *reinterpret_cast<const float4*>(&qs[p][tr * 4]);
            const float4 k0 = *reinterpret_cast<const float4*>(&ks[p][tk * 4]);
            const float4 k1 = *reinterpret_cast<const float4*>(&ks[p][64 + tk * 4]);
            const float qa[4] = {qv.x, qv.y, qv.z, qv.w};
            const float kb[8] = {k0.x, k0.y, k0.z, k0.w, k1.x, k1.y, k1.z, k1.w};
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 8; ++b) acc[a][b] = __fadd_rn(acc[a][b], __fmul_rn(qa[a], kb[b]));
        }
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const int r = r_base + tr * 4 + a;
        const int allowed = L - lq + r + 1;
        const size_t lrow = (size_t)(h - head_begin) * lq + r;
        float* out = Lp ? logits + lrow * Lp : logits + ((size_t)h * lq + r) * L;
        float m = -INFINITY;
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            const int j = j0 + (b < 4 ? tk * 4 + b : 64 + tk * 4 + (b - 4));
            const float x = __fmul_rn(acc[a][b], inv_sqrt_d);
            if (r < lq && j < allowed) {
                out[j] = x;
                m = fmaxf(m, x);
            }
        }
        if (rowmax) {  // the 16 key groups of this row sit in one half-warp
#pragma unroll
            for (int o = 1; o < 16; o <<= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
            if (tk == 0 && r < lq && m != -INFINITY) atomicMax(rowmax + lrow, enc_max(m));
        }
    }
}

// One warp per (head, row): max, e = expf(x - max) (glibc's), the sequential
// f32 sum in j order (chain_sum.cuh: exact, without the L-long chain), then
// divide.  Masked entries (j >= allowed) untouched.
__global__ void __launch_bounds__(256) score_softmax_ref(float* __restrict__ logits, int L, int lq,
                                                         int head_begin, int n_rows) {
    __shared__ uint64_t tab[32];
    tsa_dev::exp2f_table_to_smem(tab);
    __syncthreads();
    const int warp = blockIdx.x * 8 + threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    if (warp >= n_rows) return;
    const int hl = warp / lq, r = warp % lq;
    const int h = head_begin + hl;
    float* row = logits + ((size_t)h * lq + r) * L;
    const int allowed = L - lq + r + 1;
    float mx = -INFINITY;
    for (int j = lane; j < allowed; j += 32) mx = fmaxf(mx, row[j]);
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    for (int j = lane; j < allowed; j += 32) row[j] = tsa_dev::expf_glibc(__fsub_rn(row[j], mx), tab);
    __syncwarp();
    // the sequential f32 sum in j order, bit for bit, without the L-long chain
    const float sum = tsa_dev::warp_exact_chain_sum(row, allowed);
    for (int j = lane; j < allowed; j += 32) row[j] = __fdiv_rn(row[j], sum);
}

// Eigen SSE2 segment sum order (see oracle/tsa_oracle.c eigen_segment_sum).
__device__ __forceinline__ float eigen_segment_sum(const float* seg, int n, int base) {
    int a = (4 - (base & 3)) & 3;
    if (a > n) a = n;
    const int aligned_size = ((n - a) / 4) * 4;
    if (aligned_size == 0) {
        float r = seg[0];
        for (int i = 1; i < n; ++i) r = __fadd_rn(r, seg[i]);
        return r;
    }
    float p0[4], p1[4];
    for (int l = 0; l < 4; ++l) p0[l] = seg[a + l];
    const int aligned_end = a + aligned_size;
    if (aligned_size > 4) {
        const int aligned_end2 = a + ((n - a) / 8) * 8;
        for (int l = 0; l < 4; ++l) p1[l] = seg[a + 4 + l];
        for (int i = a + 8; i < aligned_end2; i += 8) {
            for (int l = 0; l < 4; ++l) p0[l] = __fadd_rn(p0[l], seg[i + l]);
            for (int l = 0; l < 4; ++l) p1[l] = __fadd_rn(p1[l], seg[i + 4 + l]);
        }
        for (int l = 0; l < 4; ++l) p0[l] = __fadd_rn(p0[l], p1[l]);
        if (aligned_end > aligned_end2)
            for (int l = 0; l < 4; ++l) p0[l] = __fadd_rn(p0[l], seg[aligned_end2 + l]);
    }
    float r = __fadd_rn(__fadd_rn(p0[0], p0[2]), __fadd_rn(p0[1], p0[3]));
    for (int i = 0; i < a; ++i) r = __fadd_rn(r, seg[i]);
    for (int i = aligned_end; i < n; ++i) r = __fadd_rn(r, seg[i]);
    return r;
}

constexpr int CS_T = 256;

// Column sums over the lq proxy rows (r ascending) for a tile of tokens plus a
// halo, then the edge-clamped pool.  Shared by REFERENCE and FAST modes:
// P rows are read from `probs` [H x lq x L] (entries past the causal limit are
// treated as exact zeros, as the reference's masked softmax writes them).
__global__ void __launch_bounds__(CS_T) score_colsum_pool(const float* __restrict__ probs,
                                                          const OutReplicas s, int L, int lq,
                                                          int kernel, int head_begin) {
    extern __shared__ float col[];  // CS_T + kernel - 1
    const int h = head_begin + blockIdx.y;
    const int t0 = blockIdx.x * CS_T;
    const int half = kernel / 2;
    const float* P = probs + (size_t)h * lq * L;
    for (int i = threadIdx.x; i < CS_T + 2 * half; i += CS_T) {
        const int t = t0 - half + i;
        float c = 0.0f;
        if (t >= 0 && t < L) {
            // row r allows t iff t <= L - lq + r  <=>  r >= t - (L - lq)
            const int r_first = max(0, t - (L - lq));
            for (int r = r_first; r < lq; ++r) c = __fadd_rn(c, P[(size_t)r * L + t]);
        }
        col[i] = c;
    }
    __syncthreads();
    const int t = t0 + threadIdx.x;
    if (t >= L) return;
    float out;
    if (kernel == 1) {
        out = col[threadIdx.x + half];
    } else {
        const int lo = max(0, t - half), hi = min(L - 1, t + half);
        const int cnt = hi - lo + 1;
        out = __fdiv_rn(eigen_segment_sum(col + (lo - t0 + half), cnt, lo), (float)cnt);
    }
    // every replica of the score rows (multi-GPU: each rank's [H x L] buffer,
    // the score all-gather fused into the producing kernel)
#pragma unroll
    for (int i = 0; i < TSA_MAX_REPLICAS; ++i) {
        if (i >= s.n) break;
        static_cast<float*>(s.p[i])[(size_t)h * L + t] = out;
    }
    if (s.n > 1) __threadfence_system();
}

}  // namespace

int launch_colsum_pool(const tsa_desc& d, const float* probs, const OutReplicas& s,
                       cudaStream_t st) {
    const int L = d.seq_len, lq = lq_of(d);
    const int nh = d.head_end - d.head_begin;
    dim3 grid((L + CS_T - 1) / CS_T, nh);
    const size_t smem = sizeof(float) * (CS_T + d.kernel - 1);
    score_colsum_pool<<<grid, CS_T, smem, st>>>(probs, s, L, lq, d.kernel, d.head_begin);
    TSA_LAUNCH_CHECK("score_colsum_pool");
    return 0;
}

int launch_score_reference(const tsa_desc& d, const void* q, const void* k, const OutReplicas& s,
                           float* logits, int* rowmax, float* rowsum, float* colraw,
                           cudaStream_t st) {
    const int L = d.seq_len, lq = lq_of(d), D = d.d_head;
    const int nh = d.head_end - d.head_begin;
    const int group = d.n_heads / d.n_kv_heads;
    const float inv_sqrt_d = 1.0f / sqrtf((float)D);
    // the exact scorer's row / column passes take these logits too (its layout
    // and row maxima); lq > 2048 keeps the per-row warp softmax
    const bool exact_rows = lq <= 2048;
    const int Lp = exact_rows ? (int)exact_logits_stride(L) : 0;
    int* rm = exact_rows ? rowmax : nullptr;
    const int n_rows = nh * lq;
    if (rm)
        if (int rc = launch_fill_int(rm, INT_MIN, n_rows, st)) return rc;
    dim3 grid((L + LG_KEYS - 1) / LG_KEYS, nh, (lq + LG_ROWS - 1) / LG_ROWS);
    if (d.dtype == TSA_BF16)
        score_logits_ref<__nv_bfloat16><<<grid, 256, 0, st>>>(
            (const __nv_bfloat16*)q, (const __nv_bfloat16*)k, logits, d.n_heads, group, L, D, lq,
            d.head_begin, inv_sqrt_d, Lp, rm);
    else
        score_logits_ref<float><<<grid, 256, 0, st>>>((const float*)q, (const float*)k, logits,
                                                      d.n_heads, group, L, D, lq, d.head_begin,
                                                      inv_sqrt_d, Lp, rm);
    TSA_LAUNCH_CHECK("score_logits_ref");
    if (exact_rows) return launch_score_exact_rows(d, logits, rm, rowsum, colraw, s, st);
    score_softmax_ref<<<(n_rows + 7) / 8, 256, 0, st>>>(logits, L, lq, d.head_begin, n_rows);
    TSA_LAUNCH_CHECK("score_softmax_ref");
    return launch_colsum_pool(d, logits, s, st);
}

}  // namespace tsa
