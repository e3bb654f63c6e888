// K5: causal flash attention on the 5th-generation tensor cores (sm_100a).
//
// dense_causal_attention (attention.cpp:25-40) -- the `inner` kernel the
// reference applies to the compressed Q^/K^/V^ of each head -- for bf16 and
// d = 128, one 128-row query tile per CTA:
//
//   warp 0      TMA producer: Q tile once, then K/V tiles through an NS-stage ring
//   warp 1      MMA issuer (one thread): S_j = Q K_j^T (SS, both K-major SW128)
//               into TMEM buffer j%2, then O += P_{j-1} V_{j-1} (TS: P read
//               from TMEM, V MN-major SW128) so that S_j runs while the softmax
//               warps work on S_{j-1}
//   warps 2..5  softmax: thread = query row = TMEM lane; tcgen05.ld the S row,
//               causal mask on the diagonal tile, online softmax in the log2
//               domain with lazy rescaling (O is only rescaled when the running
//               max grows by more than 2^8), P written back as packed bf16 into
//               the S columns (tcgen05.st); final O / l epilogue.
//
// TMEM (512 columns): S0 [0,128) S1 [128,256) O [256,384).
// n (rows per head) is read from device memory (k_keep): the grid is sized for
// L and tiles past n exit before allocating anything.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "common.cuh"
#include "sm100.cuh"

namespace tsa {
namespace {

using namespace tsa_dev;

constexpr int BM = 128;         // query rows per CTA
constexpr int BN = 128;         // keys per KV tile
constexpr int HD = 128;         // head dim
constexpr int NS = 2;           // K/V pipeline stages
constexpr int TILE_BYTES = BM * HD * 2;   // 32 KiB (two 64-col SW128 halves of 16 KiB)
constexpr int HALF_BYTES = TILE_BYTES / 2;
constexpr float kRescaleThreshold = 8.0f; // log2 units

struct __align__(1024) AttnSmem {
    uint8_t q[TILE_BYTES];
    uint8_t k[NS][TILE_BYTES];
    uint8_t v[NS][TILE_BYTES];
    uint64_t q_full;
    uint64_t k_full[NS];
    uint64_t v_full[NS];
    uint64_t kv_empty[NS];
    uint64_t s_full[2];
    uint64_t p_full[2];
    uint64_t o_done[2];
    uint32_t tmem_base;
};

__global__ void __launch_bounds__(192, 1)
attend_sm100_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_v, const int32_t* __restrict__ n_dev,
                    int n_const, int kv_group, int rows_per_head, int kv_rows_per_head,
                    int head_begin, float scale_log2, __nv_bfloat16* __restrict__ o) {
    extern __shared__ uint8_t smem_raw[];
    AttnSmem& sm = *reinterpret_cast<AttnSmem*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));

    const int h = head_begin + blockIdx.y;
    const int n = n_dev ? *n_dev : n_const;
    const int n_tiles = (n + BM - 1) / BM;
    if ((int)blockIdx.x >= n_tiles) return;
    const int mt = n_tiles - 1 - (int)blockIdx.x;  // longest causal rows first
    const int nkv = mt + 1;                          // KV tiles 0..mt
    const int kvh = h / kv_group;
    const int q_row0 = h * rows_per_head + mt * BM;
    const int kv_row0 = kvh * kv_rows_per_head;

    const uint32_t warp = warp_id_uniform();
    const uint32_t lane = lane_id();

    if (threadIdx.x == 0) {
        mbar_init(&sm.q_full, 1);
        for (int s = 0; s < NS; ++s) {
            mbar_init(&sm.k_full[s], 1);
            mbar_init(&sm.v_full[s], 1);
            mbar_init(&sm.kv_empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&sm.s_full[b], 1);
            mbar_init(&sm.p_full[b], 128);
            mbar_init(&sm.o_done[b], 1);
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(&sm.tmem_base, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sm.tmem_base;
    const uint32_t t_s[2] = {tmem, tmem + 128};
    const uint32_t t_o = tmem + 256;

    if (warp == 0) {
        // ------------------------------------------------------ TMA producer
        if (lane == 0) {
            tma_load_2d(sm.q, &tm_q, &sm.q_full, 0, q_row0);
            tma_load_2d(sm.q + HALF_BYTES, &tm_q, &sm.q_full, 64, q_row0);
            mbar_arrive_expect_tx(&sm.q_full, TILE_BYTES);
            for (int j = 0; j < nkv; ++j) {
                const int st = j % NS;
                if (j >= NS) mbar_wait(&sm.kv_empty[st], ((j / NS) - 1) & 1);
                const int r = kv_row0 + j * BN;
                tma_load_2d(sm.k[st], &tm_k, &sm.k_full[st], 0, r);
                tma_load_2d(sm.k[st] + HALF_BYTES, &tm_k, &sm.k_full[st], 64, r);
                mbar_arrive_expect_tx(&sm.k_full[st], TILE_BYTES);
                tma_load_2d(sm.v[st], &tm_v, &sm.v_full[st], 0, r);
                tma_load_2d(sm.v[st] + HALF_BYTES, &tm_v, &sm.v_full[st], 64, r);
                mbar_arrive_expect_tx(&sm.v_full[st], TILE_BYTES);
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------ MMA issuer
        if (lane == 0) {
            const uint32_t idesc_s = idesc_bf16_f32(BM, BN, 0, 0);
            const uint32_t idesc_o = idesc_bf16_f32(BM, HD, 0, 1);
            const uint32_t q_base = smem_u32(sm.q);
            mbar_wait(&sm.q_full, 0);
            tc_fence_after();
            auto issue_pv = [&](int j) {
                const int st = j % NS, b = j & 1;
                mbar_wait(&sm.p_full[b], (j >> 1) & 1);
                mbar_wait(&sm.v_full[st], (j / NS) & 1);
                tc_fence_after();
                const uint32_t v_base = smem_u32(sm.v[st]);
#pragma unroll
                for (int kk = 0; kk < BN / 16; ++kk)
                    mma_bf16_ts(t_o, t_s[b] + kk * 8, sdesc_mnmajor_sw128(v_base + kk * 2048, HALF_BYTES),
                                idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
                mma_commit(&sm.o_done[b]);
                mma_commit(&sm.kv_empty[st]);
            };
            for (int j = 0; j < nkv; ++j) {
                const int st = j % NS, b = j & 1;
                mbar_wait(&sm.k_full[st], (j / NS) & 1);
                tc_fence_after();
                const uint32_t k_base = smem_u32(sm.k[st]);
#pragma unroll
                for (int kk = 0; kk < HD / 16; ++kk) {
                    const uint32_t off = (kk >> 2) * HALF_BYTES + (kk & 3) * 32;
                    mma_bf16_ss(t_s[b], sdesc_kmajor_sw128(q_base + off),
                                sdesc_kmajor_sw128(k_base + off), idesc_s, kk > 0 ? 1u : 0u);
                }
                mma_commit(&sm.s_full[b]);
                if (j >= 1) issue_pv(j - 1);
            }
            issue_pv(nkv - 1);
        }
    } else {
        // ------------------------------------------------------ softmax warps
        const uint32_t sub = warp & 3;           // TMEM lane sub-partition of this warp
        const int row = (int)(sub * 32 + lane);  // query row within the tile
        const int qi = mt * BM + row;            // compressed row index
        const uint32_t lane_off = (sub * 32) << 16;
        float m_run = -INFINITY, l_run = 0.0f;
        for (int j = 0; j < nkv; ++j) {
            const int b = j & 1;
            mbar_wait(&sm.s_full[b], (j >> 1) & 1);
            tc_fence_after();
            float s[BN];
#pragma unroll
            for (int c = 0; c < BN; c += 32) {
                uint32_t r[32];
                tmem_ld32(t_s[b] + lane_off + c, r);
                tmem_wait_ld();
#pragma unroll
                for (int e = 0; e < 32; ++e) s[c + e] = __uint_as_float(r[e]);
            }
            const bool diag = (j == mt);
            float tmax = -INFINITY;
#pragma unroll
            for (int c = 0; c < BN; ++c) {
                float x = s[c] * scale_log2;
                if (diag && (j * BN + c) > qi) x = -INFINITY;
                s[c] = x;
                tmax = fmaxf(tmax, x);
            }
            // lazy rescale: only move the reference max when it grows by > 2^8
            float m_use = m_run;
            bool rescale = false;
            if (tmax > m_run + kRescaleThreshold || m_run == -INFINITY) {
                m_use = tmax;
                rescale = (j > 0) && (m_run != -INFINITY);
            }
            if (m_use == -INFINITY) m_use = 0.0f;  // fully masked row (rows >= n)
            // P_j reuses S buffer b: P_{j-2} must have been consumed (PV_{j-2} done)
            if (j >= 2) {
                mbar_wait(&sm.o_done[b], ((j - 2) >> 1) & 1);
            }
            float lsum = 0.0f;
            uint32_t packed[BN / 2];
#pragma unroll
            for (int c = 0; c < BN; c += 2) {
                const float p0 = ex2_approx(s[c] - m_use);
                const float p1 = ex2_approx(s[c + 1] - m_use);
                lsum += p0 + p1;
                packed[c / 2] = pack_bf16x2(p0, p1);
            }
            // tcgen05.ld/st are warp-collective (.sync.aligned): the whole warp
            // rescales when any of its rows needs it (alpha = 1 for the others)
            if (__any_sync(0xffffffffu, rescale)) {
                // O must hold PV_{j-1} before it is rescaled
                mbar_wait(&sm.o_done[b ^ 1], ((j - 1) >> 1) & 1);
                tc_fence_after();
                const float alpha = rescale ? ex2_approx(m_run - m_use) : 1.0f;
#pragma unroll
                for (int c = 0; c < HD; c += 32) {
                    uint32_t r[32];
                    tmem_ld32(t_o + lane_off + c, r);
                    tmem_wait_ld();
#pragma unroll
                    for (int e = 0; e < 32; ++e) r[e] = __float_as_uint(__uint_as_float(r[e]) * alpha);
                    tmem_st32(t_o + lane_off + c, r);
                }
                if (rescale) l_run *= alpha;
            }
            l_run += lsum;
            m_run = m_use;
#pragma unroll
            for (int c = 0; c < BN / 2; c += 32) {
                uint32_t r[32];
#pragma unroll
                for (int e = 0; e < 32; ++e) r[e] = packed[c + e];
                tmem_st32(t_s[b] + lane_off + c, r);
            }
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(&sm.p_full[b]);
        }
        // epilogue: O / l -> bf16 -> global (thread writes its 256-B row)
        const int jl = nkv - 1;
        mbar_wait(&sm.o_done[jl & 1], (jl >> 1) & 1);
        tc_fence_after();
        const float inv_l = 1.0f / l_run;
        __nv_bfloat16* dst = o + ((size_t)q_row0 + row) * HD;
#pragma unroll
        for (int c = 0; c < HD; c += 32) {
            uint32_t r[32];
            tmem_ld32(t_o + lane_off + c, r);
            tmem_wait_ld();
            if (qi < n) {
                uint4 outv[4];
                uint32_t* ow = reinterpret_cast<uint32_t*>(outv);
#pragma unroll
                for (int e = 0; e < 16; ++e)
                    ow[e] = pack_bf16x2(__uint_as_float(r[2 * e]) * inv_l,
                                        __uint_as_float(r[2 * e + 1]) * inv_l);
                uint4* d4 = reinterpret_cast<uint4*>(dst + c);
#pragma unroll
                for (int e = 0; e < 4; ++e) d4[e] = outv[e];
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, 512);
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

bool attend_sm100_supported(const tsa_desc& d) { return d.dtype == TSA_BF16 && d.d_head == HD; }

int launch_attend_sm100(const tsa_desc& d, const void* q, const void* k, const void* v,
                        const int32_t* n_dev, int32_t n_const, int32_t kv_group,
                        int32_t rows_per_head, int32_t kv_rows_per_head, void* o,
                        cudaStream_t st) {
    if (!attend_sm100_supported(d)) return invalid("attend_sm100: needs bf16, d_head 128");
    const int nh = d.head_end - d.head_begin;
    const int n_q_heads = d.n_heads;
    const int n_kv_heads_buf = (n_q_heads + kv_group - 1) / kv_group;
    CUtensorMap mq, mk, mv;
    int rc;
    if ((rc = make_bf16_map_2d(&mq, q, (uint64_t)n_q_heads * rows_per_head, 128))) return rc;
    if ((rc = make_bf16_map_2d(&mk, k, (uint64_t)n_kv_heads_buf * kv_rows_per_head, 128))) return rc;
    if ((rc = make_bf16_map_2d(&mv, v, (uint64_t)n_kv_heads_buf * kv_rows_per_head, 128))) return rc;
    const int smem = (int)sizeof(AttnSmem) + 1024;
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(attend_sm100_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        attr_set = true;
    }
    dim3 grid((rows_per_head + BM - 1) / BM, nh);
    const float scale_log2 = (1.0f / sqrtf((float)HD)) * 1.4426950408889634f;
    attend_sm100_kernel<<<grid, 192, smem, st>>>(mq, mk, mv, n_dev, n_const, kv_group, rows_per_head,
                                                 kv_rows_per_head, d.head_begin, scale_log2,
                                                 (__nv_bfloat16*)o);
    TSA_LAUNCH_CHECK("attend_sm100");
    return 0;
}

}  // namespace tsa
