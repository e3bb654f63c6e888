// The attention branch's projections on the 5th-generation tensor cores
// (layer_forward, model.cpp:169-201), with the work around them fused into
// the GEMM epilogues:
//
//   QKV   q, k, v = split_heads(rope(rms_norm(x) W_qkv))     model.cpp:81-94, 107-158
//         A = x [L][D] as stored; rms_norm's per-row 1/rms scales the
//         accumulator (the gain vector is folded into W once: prepare_weight),
//         RoPE rotates the q / k columns in f32 and the rows go straight to
//         q [H][L][d], k / v [Hkv][L][d] -- no normalised copy of x, no
//         projection buffer, no split pass.
//   OUT   x += concat_h(o_h) W_o                             model.cpp:196-201
//         A is read from the attention output o [H][L][d] through a 3-D
//         tensor map (the K index h*d + j walks the heads), so the head concat
//         is never materialised; the residual add is the epilogue.
//   STORE c = a b^T (the plain GEMM, for tests and comparisons).
//
// One persistent kernel over 256 x 256 output tiles, run by CTA PAIRS
// (2-CTA clusters, cta_group::2): each CTA stages its 128 rows of A and its
// 128 rows of B (K-major, W stored transposed [N][K]) per 64-wide K step
// through a 6-stage TMA ring (16 + 16 KiB, 128-B swizzle), and the leader CTA
// issues M256 N256 K16 MMAs that read both CTAs' shared memory, so every
// operand byte staged feeds twice the MMA work of a one-CTA tile:
//   warp 0        TMA producer (both CTAs; completion bytes on the leader's barrier)
//   warp 1        MMA issuer (leader CTA): 4 MMAs per stage into one of two TMEM
//                 accumulators (2 x 256 columns in each CTA), so the epilogue
//                 of tile i overlaps the main loop of tile i+1; commits are
//                 multicast to both CTAs
//   warps 2..9    epilogue (both CTAs): thread = output row = TMEM lane, two
//                 warps per lane quarter with four 32-column chunks each
//                 (tcgen05.ld) -> fused op -> 16-B stores; the chunk's global
//                 inputs (residual, RoPE angles) are loaded ahead of it;
//                 the accumulator is handed back on the leader's barrier
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "sm100.cuh"

namespace tsa {

int make_bf16_map_3d(CUtensorMap* m, const void* base, uint64_t rows, uint64_t heads);
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder();

namespace {

using namespace tsa_dev;

constexpr int GM = 256;   // output rows per pair tile (128 per CTA)
constexpr int GN = 256;   // output columns per tile
constexpr int CM = 128;   // A rows per CTA
constexpr int CN = 128;   // B rows (output columns) staged per CTA
constexpr int GK = 64;    // K per stage (one 128-B swizzle row of bf16)
constexpr int GS = 6;     // ring stages
constexpr int A_BYTES = CM * GK * 2;
constexpr int B_BYTES = CN * GK * 2;
constexpr int kGemmThreads = 320;  // producer, MMA, 8 epilogue warps
constexpr int kChunksPerWarp = GN / 32 / 2;
constexpr int kHeadDim = 128;  // QKV / OUT epilogues: d_head

enum Epi { kEpiStore = 0, kEpiQkv = 1, kEpiResid = 2 };

struct __align__(1024) GemmSmem {
    uint8_t a[GS][A_BYTES];
    uint8_t b[GS][B_BYTES];
    uint64_t full[GS], empty[GS], acc_full[2], acc_empty[2];
    uint32_t tmem_base;
};

struct EpiArgs {
    void* c;                   // STORE: c [M][ldc]; RESID: x [M][ldc] (read-modify-write)
    int64_t ldc;
    const float* inv_rms;      // QKV: per-row 1/rms (nullptr: no norm)
    const float4* table;       // QKV: RoPE table [L][d/2] of (cos, sin) pairs, 2 pairs per float4
    __nv_bfloat16* q;          // QKV outputs
    __nv_bfloat16* k;
    __nv_bfloat16* v;
    int n_q_heads, n_kv_heads;
};

// Shared-memory descriptor low word (start address >> 4, LBO 16 B); the high
// word (SBO 1 KiB = 8 swizzled 128-B rows, version 1, SWIZZLE_128B) is constant.
__device__ __forceinline__ uint64_t gdesc(uint32_t saddr) {
    return (static_cast<uint64_t>(0x40004040u) << 32) | (((saddr >> 4) & 0x3FFFu) | (1u << 16));
}

__device__ __forceinline__ void store_row32(__nv_bfloat16* dst, const float (&v)[32]) {
    uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
    for (int u = 0; u < 4; ++u)
        d4[u] = make_uint4(pack_bf16x2(v[8 * u + 0], v[8 * u + 1]), pack_bf16x2(v[8 * u + 2], v[8 * u + 3]),
                           pack_bf16x2(v[8 * u + 4], v[8 * u + 5]), pack_bf16x2(v[8 * u + 6], v[8 * u + 7]));
}

// The epilogue's global inputs for 32 columns [n, n + 32) of output row `row`
// (the residual row slice, or the RoPE angles), loaded BEFORE the chunk's
// tcgen05.ld so the two latencies overlap.
struct ChunkAux {
    uint4 u[8];
};

template <int kEpi>
__device__ __forceinline__ void epilogue_aux(const EpiArgs& e, int64_t row, int n, ChunkAux& a) {
    if constexpr (kEpi == kEpiResid) {
        const uint4* x4 = reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(e.c) +
                                                         row * e.ldc + n);
#pragma unroll
        for (int u = 0; u < 4; ++u) a.u[u] = x4[u];
    } else if constexpr (kEpi == kEpiQkv) {
        const int slot = n / kHeadDim, c0 = n % kHeadDim;
        if (slot < e.n_q_heads + e.n_kv_heads) {
            // pairs (c0/2 .. c0/2 + 15) of position `row`: 8 float4 of (cos, sin, cos, sin)
            const uint4* tb = reinterpret_cast<const uint4*>(e.table + (row * (kHeadDim / 2) + c0 / 2) / 2);
#pragma unroll
            for (int u = 0; u < 8; ++u) a.u[u] = __ldg(tb + u);
        }
    }
}

// 32 accumulator columns [n, n + 32) of output row `row`.
template <int kEpi>
__device__ __forceinline__ void epilogue_chunk(const EpiArgs& e, const uint32_t (&r)[32], int64_t row,
                                               int n, int L, float row_scale, const ChunkAux& a) {
    float v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
    if constexpr (kEpi == kEpiStore) {
        store_row32(reinterpret_cast<__nv_bfloat16*>(e.c) + row * e.ldc + n, v);
    } else if constexpr (kEpi == kEpiResid) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const __nv_bfloat162* p2 = reinterpret_cast<const __nv_bfloat162*>(&a.u[u]);
#pragma unroll
            for (int w = 0; w < 4; ++w) {
                const float2 f = __bfloat1622float2(p2[w]);
                v[8 * u + 2 * w] = __fadd_rn(f.x, v[8 * u + 2 * w]);
                v[8 * u + 2 * w + 1] = __fadd_rn(f.y, v[8 * u + 2 * w + 1]);
            }
        }
        store_row32(reinterpret_cast<__nv_bfloat16*>(e.c) + row * e.ldc + n, v);
    } else {  // kEpiQkv: rms scale, RoPE on q / k, head split
        if (e.inv_rms) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = __fmul_rn(v[j], row_scale);
        }
        const int slot = n / kHeadDim, c0 = n % kHeadDim;
        const int hq = e.n_q_heads, hk = e.n_kv_heads;
        if (slot < hq + hk) {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const float4 cs = *reinterpret_cast<const float4*>(&a.u[u]);
                float x0 = v[4 * u], x1 = v[4 * u + 1];
                v[4 * u] = __fsub_rn(__fmul_rn(x0, cs.x), __fmul_rn(x1, cs.y));
                v[4 * u + 1] = __fadd_rn(__fmul_rn(x0, cs.y), __fmul_rn(x1, cs.x));
                x0 = v[4 * u + 2];
                x1 = v[4 * u + 3];
                v[4 * u + 2] = __fsub_rn(__fmul_rn(x0, cs.z), __fmul_rn(x1, cs.w));
                v[4 * u + 3] = __fadd_rn(__fmul_rn(x0, cs.w), __fmul_rn(x1, cs.z));
            }
        }
        __nv_bfloat16* dst = slot < hq        ? e.q + ((int64_t)slot * L + row) * kHeadDim
                             : slot < hq + hk ? e.k + ((int64_t)(slot - hq) * L + row) * kHeadDim
                                              : e.v + ((int64_t)(slot - hq - hk) * L + row) * kHeadDim;
        store_row32(dst + c0, v);
    }
}

template <int kEpi, bool kA3D>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kGemmThreads, 1)
proj_gemm_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                 int M, int N, int K, const __grid_constant__ EpiArgs e) {
    extern __shared__ uint8_t smem_raw[];
    GemmSmem& sm = *reinterpret_cast<GemmSmem*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t warp = warp_id_uniform();
    const uint32_t lane = lane_id();
    const uint32_t rank = cluster_ctarank();
    const int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;
    const int n_blocks = N / GN;
    const int n_tiles = ((M + GM - 1) / GM) * n_blocks;
    const int n_kb = K / GK;

    if (threadIdx.x == 0) {
        for (int s = 0; s < GS; ++s) {
            mbar_init(&sm.full[s], 1);
            mbar_init(&sm.empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&sm.acc_full[b], 1);
            mbar_init(&sm.acc_empty[b], 16);  // one arrival per epilogue warp of both CTAs
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc_pair(&sm.tmem_base, 512);
    tc_fence_before();
    cluster_sync_all();  // barriers initialised in both CTAs before any remote arrival
    tc_fence_after();
    const uint32_t tmem = sm.tmem_base;

    if (warp == 0) {
        // ------------------------------------------------------------ TMA producer
        if (lane == 0) {
            tma_prefetch_desc(&tm_a);
            tma_prefetch_desc(&tm_b);
            uint32_t it = 0;
            for (int tile = pair; tile < n_tiles; tile += n_pairs) {
                const int m0 = (tile / n_blocks) * GM + (int)rank * CM;
                const int n0 = (tile % n_blocks) * GN + (int)rank * CN;
                for (int kb = 0; kb < n_kb; ++kb, ++it) {
                    const uint32_t s = it % GS;
                    if (it >= GS) mbar_wait(&sm.empty[s], ((it / GS) - 1) & 1);
                    if (rank == 0) mbar_arrive_expect_tx(&sm.full[s], 2 * (A_BYTES + B_BYTES));
                    if constexpr (kA3D) {  // A[m][h d + j] = o[h][m][j]
                        const int kk = kb * GK;
                        tma_load_3d_pair(sm.a[s], &tm_a, &sm.full[s], kk % kHeadDim, m0, kk / kHeadDim);
                    } else {
                        tma_load_2d_pair(sm.a[s], &tm_a, &sm.full[s], kb * GK, m0);
                    }
                    tma_load_2d_pair(sm.b[s], &tm_b, &sm.full[s], kb * GK, n0);
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        if (rank == 0) {
            const uint32_t issue = elect_one() ? 1u : 0u;
            constexpr uint32_t idesc = idesc_bf16_f32(GM, GN, 0, 0);
            uint32_t it = 0, local = 0;
            for (int tile = pair; tile < n_tiles; tile += n_pairs, ++local) {
                const uint32_t b = local & 1, use = local >> 1;
                if (local >= 2) mbar_wait(&sm.acc_empty[b], (use - 1) & 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem + b * GN;
                for (int kb = 0; kb < n_kb; ++kb, ++it) {
                    const uint32_t s = it % GS;
                    mbar_wait(&sm.full[s], (it / GS) & 1);
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(sm.a[s]), b0 = smem_u32(sm.b[s]);
#pragma unroll
                    for (int kk = 0; kk < GK / 16; ++kk)
                        mma_bf16_ss_pair_p(d_tmem, gdesc(a0 + kk * 32), gdesc(b0 + kk * 32), idesc,
                                           (kb | kk) ? 1u : 0u, issue);
                    mma_commit_pair_p(&sm.empty[s], issue);
                }
                mma_commit_pair_p(&sm.acc_full[b], issue);
            }
        }
    } else {
        // ------------------------------------------------------------ epilogue
        // two warps per TMEM lane quarter, each four of the eight 32-column chunks
        const uint32_t quarter = warp & 3;  // TMEM lane quarter this warp may access
        const int c_begin = warp < 6 ? 0 : kChunksPerWarp;
        uint32_t local = 0;
        for (int tile = pair; tile < n_tiles; tile += n_pairs, ++local) {
            const uint32_t b = local & 1, use = local >> 1;
            const int m0 = (tile / n_blocks) * GM + (int)rank * CM, n0 = (tile % n_blocks) * GN;
            const int64_t row = m0 + (int)(quarter * 32 + lane);
            const bool live = row < M;
            const float row_scale = (kEpi == kEpiQkv && e.inv_rms && live) ? __ldg(e.inv_rms + row) : 1.0f;
            ChunkAux aux;
            if (live) epilogue_aux<kEpi>(e, row, n0 + c_begin * 32, aux);
            mbar_wait(&sm.acc_full[b], use & 1);
            tc_fence_after();
            const uint32_t taddr = tmem + ((quarter * 32) << 16) + b * GN;
#pragma unroll 1
            for (int c = c_begin; c < c_begin + kChunksPerWarp; ++c) {
                uint32_t r[32];
                tmem_ld32(taddr + c * 32, r);
                tmem_wait_ld();
                if (c == c_begin + kChunksPerWarp - 1) {  // drained: the MMA may reuse it
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_leader(&sm.acc_empty[b]);
                }
                if (live) {
                    epilogue_chunk<kEpi>(e, r, row, n0 + c * 32, M, row_scale, aux);
                    if (c + 1 < c_begin + kChunksPerWarp) epilogue_aux<kEpi>(e, row, n0 + (c + 1) * 32, aux);
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();  // the leader's MMAs into this CTA's TMEM / smem are complete
    tc_fence_after();
    if (warp == 1) tmem_dealloc_pair(tmem, 512);
}

// [rows][inner] bf16, K-major boxes of 64 x box_rows, 128-B swizzle.
int make_kmajor_map(CUtensorMap* m, const void* base, uint64_t inner, uint64_t rows,
                    uint32_t box_rows) {
    auto fn = tensor_map_encoder();
    if (!fn) return invalid("tsa: cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {inner, rows};
    cuuint64_t strides[1] = {inner * 2};
    cuuint32_t box[2] = {GK, box_rows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                    box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        return invalid("tsa: GEMM tensor map encode failed (" + std::to_string((int)r) + ")");
    return 0;
}

template <int kEpi, bool kA3D>
int run_gemm(const CUtensorMap& ma, const CUtensorMap& mb, int M, int N, int K, const EpiArgs& e,
             cudaStream_t st) {
    const int smem = (int)sizeof(GemmSmem) + 1024;
    auto fn = proj_gemm_kernel<kEpi, kA3D>;
    if (int rc = ensure_smem_attr(reinterpret_cast<const void*>(fn), smem)) return rc;
    const int n_tiles = ((M + GM - 1) / GM) * (N / GN);
    const int pairs = n_tiles < num_sms() / 2 ? n_tiles : num_sms() / 2;
    fn<<<2 * pairs, kGemmThreads, smem, st>>>(ma, mb, M, N, K, e);
    TSA_LAUNCH_CHECK("proj_gemm");
    return 0;
}

// ---- small HBM-bound helpers

// inv[r] = 1 / sqrt(sum_j x[r, j]^2 / cols + eps): one warp per row, 16-B loads.
__global__ void __launch_bounds__(256) row_inv_rms_kernel(const __nv_bfloat16* __restrict__ x,
                                                         int64_t rows, int cols, float eps,
                                                         float* __restrict__ inv) {
    const int64_t r = (int64_t)blockIdx.x * 8 + threadIdx.x / 32;
    if (r >= rows) return;
    const int lane = threadIdx.x & 31;
    const uint4* row = reinterpret_cast<const uint4*>(x + r * cols);
    float acc = 0.0f;
    for (int u = lane; u < cols / 8; u += 32) {
        const uint4 raw = __ldg(row + u);
        const __nv_bfloat162* p2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            const float2 f = __bfloat1622float2(p2[w]);
            acc = fmaf(f.x, f.x, acc);
            acc = fmaf(f.y, f.y, acc);
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) inv[r] = 1.0f / sqrtf(acc / (float)cols + eps);
}

// w_t[n][k] = bf16(gain[k] * w[k][n]) (gain may be null): 32 x 32 tiles.
template <typename T>
__global__ void prepare_weight_kernel(const T* __restrict__ w, const float* __restrict__ gain,
                                      int rows, int cols, __nv_bfloat16* __restrict__ w_t) {
    __shared__ float tile[32][33];
    const int k0 = blockIdx.y * 32, n0 = blockIdx.x * 32;
    for (int i = threadIdx.y; i < 32; i += 8) {
        const int k = k0 + i, n = n0 + threadIdx.x;
        float val = 0.0f;
        if (k < rows && n < cols) {
            val = Elem<T>::to_f32(w[(int64_t)k * cols + n]);
            if (gain) val = __fmul_rn(val, gain[k]);
        }
        tile[i][threadIdx.x] = val;
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += 8) {
        const int n = n0 + i, k = k0 + threadIdx.x;
        if (n < cols && k < rows) w_t[(int64_t)n * rows + k] = __float2bfloat16(tile[threadIdx.x][i]);
    }
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace

int launch_gemm_bf16(const void* a, const void* b_t, void* c, int M, int N, int K, cudaStream_t st) {
    if (M < 1 || N % GN || K % GK || N < GN || K < GK)
        return invalid("gemm_bf16: needs M >= 1, N a multiple of 256, K a multiple of 64");
    if (!aligned16(a) || !aligned16(b_t) || !aligned16(c))
        return invalid("gemm_bf16: a, b_t and c must be 16-byte aligned");
    CUtensorMap ma, mb;
    int rc;
    if ((rc = make_kmajor_map(&ma, a, K, M, CM))) return rc;
    if ((rc = make_kmajor_map(&mb, b_t, K, N, CN))) return rc;
    EpiArgs e{};
    e.c = c;
    e.ldc = N;
    return run_gemm<kEpiStore, false>(ma, mb, M, N, K, e, st);
}

int launch_qkv_proj(const tsa_desc& d, const void* x, int d_model, const void* w_t,
                    const float* inv_rms, const float* table, void* q, void* k, void* v,
                    cudaStream_t st) {
    const int L = d.seq_len, N = (d.n_heads + 2 * d.n_kv_heads) * d.d_head;
    if (d.dtype != TSA_BF16 || d.d_head != kHeadDim)
        return invalid("qkv_proj: needs bf16 and d_head 128");
    if (N % GN) return invalid("qkv_proj: (H + 2 Hkv) d must be a multiple of 256");
    if (d_model % GK || d_model < GK) return invalid("qkv_proj: d_model must be a multiple of 64");
    if (!aligned16(x) || !aligned16(w_t) || !aligned16(table) || !aligned16(q) || !aligned16(k) ||
        !aligned16(v))
        return invalid("qkv_proj: x, w_t, table, q, k, v must be 16-byte aligned");
    CUtensorMap ma, mb;
    int rc;
    if ((rc = make_kmajor_map(&ma, x, d_model, L, CM))) return rc;
    if ((rc = make_kmajor_map(&mb, w_t, d_model, N, CN))) return rc;
    EpiArgs e{};
    e.inv_rms = inv_rms;
    e.table = reinterpret_cast<const float4*>(table);
    e.q = static_cast<__nv_bfloat16*>(q);
    e.k = static_cast<__nv_bfloat16*>(k);
    e.v = static_cast<__nv_bfloat16*>(v);
    e.n_q_heads = d.n_heads;
    e.n_kv_heads = d.n_kv_heads;
    return run_gemm<kEpiQkv, false>(ma, mb, L, N, d_model, e, st);
}

int launch_out_proj_residual(const tsa_desc& d, const void* o, const void* wo_t, int d_model,
                             void* x, cudaStream_t st) {
    const int L = d.seq_len, K = d.n_heads * d.d_head;
    if (d.dtype != TSA_BF16 || d.d_head != kHeadDim)
        return invalid("out_proj_residual: needs bf16 and d_head 128");
    if (d_model % GN || d_model < GN) return invalid("out_proj_residual: d_model must be a multiple of 256");
    if (!aligned16(o) || !aligned16(wo_t) || !aligned16(x))
        return invalid("out_proj_residual: o, wo_t and x must be 16-byte aligned");
    CUtensorMap ma, mb;
    int rc;
    if ((rc = make_bf16_map_3d(&ma, o, L, d.n_heads))) return rc;  // 64 x 128 x 1 SW128 boxes
    if ((rc = make_kmajor_map(&mb, wo_t, K, d_model, CN))) return rc;
    EpiArgs e{};
    e.c = x;
    e.ldc = d_model;
    return run_gemm<kEpiResid, true>(ma, mb, L, d_model, K, e, st);
}

int launch_row_inv_rms(const void* x, int64_t rows, int cols, float eps, float* inv, cudaStream_t st) {
    if (rows < 1) return 0;
    if (cols % 8 || cols < 8) return invalid("row_inv_rms: cols must be a multiple of 8");
    row_inv_rms_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(
        static_cast<const __nv_bfloat16*>(x), rows, cols, eps, inv);
    TSA_LAUNCH_CHECK("row_inv_rms");
    return 0;
}

int launch_prepare_weight(const void* w, int dtype, const float* gain, int rows, int cols, void* w_t,
                          cudaStream_t st) {
    dim3 grid((cols + 31) / 32, (rows + 31) / 32), block(32, 8);
    if (dtype == TSA_BF16)
        prepare_weight_kernel<__nv_bfloat16><<<grid, block, 0, st>>>(
            static_cast<const __nv_bfloat16*>(w), gain, rows, cols, static_cast<__nv_bfloat16*>(w_t));
    else
        prepare_weight_kernel<float><<<grid, block, 0, st>>>(static_cast<const float*>(w), gain, rows,
                                                             cols, static_cast<__nv_bfloat16*>(w_t));
    TSA_LAUNCH_CHECK("prepare_weight");
    return 0;
}

}  // namespace tsa
