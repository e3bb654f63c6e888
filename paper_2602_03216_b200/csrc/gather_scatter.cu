// K4 gather / K6 scatter: HBM-bound row movement with 16-byte vector accesses.
//
// gather  (gather_rows x3, tensor_ops.cpp:92-99 via attention.cpp:93-95):
//   qc[h, r] = q[h, idx[h, r]],  kc[h, r] = k[kv(h), idx[h, r]],  vc likewise,
//   for r < k_keep (device).  Bytes per call: 6 * H_shard * k * d * b (+ 4 * H * k idx).
// scatter (scatter_rows, tensor_ops.cpp:101-112 via attention.cpp:96):
//   out[h, t] = oc[h, inv[h, t]] if inv >= 0 else +0.0 -- every output row is
//   written exactly once (no zero-fill pass).  Bytes: H*L*d*b written +
//   H*k*d*b read + 4*H*L inv.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "sm100.cuh"

namespace tsa {

int make_bf16_rows_map(CUtensorMap* m, const void* base, uint64_t rows, uint32_t box_rows);
int make_bf16_rows_map_3d(CUtensorMap* m, const void* base, uint64_t rows, uint64_t heads,
                          uint32_t box_rows);

namespace {

// A block moves 64 rows of one head: the 64 indices are staged in shared
// memory first, then every thread copies whole access units (chunk c of row
// r) with all of its loads issued before its stores, so each thread keeps
// several independent 16-B requests in flight.
// V is the access unit: 16 B when a row is a multiple of 16 B (every
// production shape), else 4 or 2 B for the small head sizes the reference's
// unit tests use (d = 1, 4).  Rows [n, ceil128(n)) are zeroed: the
// tensor-core attention loads whole tiles, and P = 0 times a stale NaN would
// poison O.
constexpr int G_ROWS = 64;

template <typename V, int kChunks>  // kChunks: access units per row if fixed (d = 128 bf16: 16), else 0
__global__ void __launch_bounds__(256) gather_kernel(const V* __restrict__ q,
                                                     const V* __restrict__ k,
                                                     const V* __restrict__ v,
                                                     const int32_t* __restrict__ idx,
                                                     const int32_t* __restrict__ k_keep_p,
                                                     V* __restrict__ qc, V* __restrict__ kc,
                                                     V* __restrict__ vc, int L, int group,
                                                     int chunks_rt /* access units per row */,
                                                     int head_begin,
                                                     const int32_t* __restrict__ inv,
                                                     const OutReplicas out, int skip_identity) {
    __shared__ int32_t rows[G_ROWS];
    __shared__ bool drop[G_ROWS];
    // a compile-time row width turns the per-unit row / column split into shifts
    const int chunks = kChunks ? kChunks : chunks_rt;
    // block order: the `group` query heads sharing a KV head are adjacent and
    // take the same 64-row block of their selections, whose token positions
    // nearly coincide -- the K/V rows they read hit L2 after the first head
    const int nrb = gridDim.x / group;  // row blocks per head
    const int hg = blockIdx.x % group, rb = blockIdx.x / group;
    const int h = head_begin + blockIdx.y * group + hg;
    const int kv = h / group;
    const int n = *k_keep_p;
    const int r0 = rb * G_ROWS;
    (void)nrb;
    const int pad_end = min(L, (n + 127) / 128 * 128);
    // k_keep == L: the selection is the identity and the fused attention reads
    // K/V in place (attend_sm100 in_place), so the compressed copy is skipped
    const bool gather = r0 < pad_end && !(skip_identity && n == L);
    if (!gather && out.n == 0) return;
    if (threadIdx.x < G_ROWS) {
        const int r = r0 + threadIdx.x;
        rows[threadIdx.x] = gather && r < n ? idx[(size_t)h * L + r] : -1;
        // fused zero-fill: output rows the selection dropped (scatter_rows'
        // zero rows, tensor_ops.cpp:107): fire-and-forget stores beside the gather
        if (out.n) drop[threadIdx.x] = r < L && __ldg(inv + (size_t)h * L + r) < 0;
    }
    __syncthreads();
    if (out.n) {
        // every replica of the output (multi-GPU: this rank's and the peers'
        // buffers over NVLink) receives the same rows
#pragma unroll
        for (int i = 0; i < TSA_MAX_REPLICAS; ++i) {
            if (i >= out.n) break;
            V* o = static_cast<V*>(out.p[i]) + ((size_t)h * L + r0) * chunks;
            for (int e = threadIdx.x; e < G_ROWS * chunks; e += 256)
                if (drop[e / chunks]) o[e] = V{};
        }
        if (out.n > 1) __threadfence_system();
    }
    if (!gather) return;
    const int total = G_ROWS * chunks;
    constexpr int U = 4;
    for (int e0 = threadIdx.x; e0 < total; e0 += 256 * U) {
        V kb[U], vb[U], qb[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int e = e0 + u * 256;
            kb[u] = V{};
            vb[u] = V{};
            qb[u] = V{};
            if (e < total) {
                const int rr = e / chunks, c = e % chunks;
                const int t = rows[rr];
                if (t >= 0) {
                    const size_t src_kv = ((size_t)kv * L + t) * chunks + c;
                    kb[u] = __ldg(k + src_kv);
                    vb[u] = __ldg(v + src_kv);
                    if (qc) qb[u] = __ldg(q + ((size_t)h * L + t) * chunks + c);
                }
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int e = e0 + u * 256;
            if (e >= total) continue;
            const int rr = e / chunks, c = e % chunks;
            if (r0 + rr >= pad_end) continue;
            const size_t dst = ((size_t)h * L + r0 + rr) * chunks + c;
            kc[dst] = kb[u];
            vc[dst] = vb[u];
            if (qc) qc[dst] = qb[u];
        }
    }
}

// The K/V compress of the fused path (bf16, d = 128) on the TMA: per block of
// 64 compressed rows one thread issues 16 tile::gather4 loads per tensor (4
// selected rows of 256 B each) into shared memory and one bulk tensor store of
// the 64 rows (16 KB) per tensor -- the copy costs a few dozen instructions per
// 32 KB instead of two thousand 16-B loads and stores.  Rows in [n, ceil128(n))
// are read out of bounds (zeros).  The dropped output rows of the block's 64
// positions are zeroed by all threads with streaming stores beside it.
constexpr int GT_ROWS = 64;

struct __align__(128) GatherSmem {
    uint8_t k[GT_ROWS * 256];
    uint8_t v[GT_ROWS * 256];
    uint64_t full;
    int32_t rows[GT_ROWS];
    bool drop[GT_ROWS];
};

__global__ void __launch_bounds__(256) gather_tma_kernel(
    const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
    const __grid_constant__ CUtensorMap tm_kc, const __grid_constant__ CUtensorMap tm_vc,
    const int32_t* __restrict__ idx, const int32_t* __restrict__ k_keep_p, int L, int group,
    int head_begin, int kv_rows, const int32_t* __restrict__ inv, const OutReplicas out) {
    __shared__ GatherSmem sm;
    using namespace tsa_dev;
    const int hg = blockIdx.x % group, rb = blockIdx.x / group;
    const int h = head_begin + blockIdx.y * group + hg;  // kc / vc / out are indexed by h
    const int kv = h / group - head_begin / group;
    const int n = *k_keep_p;
    const int r0 = rb * GT_ROWS;
    const int pad_end = min(L, (n + 127) / 128 * 128);
    // k_keep == L: identity selection, the attention reads K/V in place
    const bool gather = r0 < pad_end && n != L;
    if (!gather && out.n == 0) return;
    const int tid = threadIdx.x;
    if (tid < GT_ROWS) {
        const int r = r0 + tid;
        // rows past k_keep read out of bounds: TMA fills zeros
        sm.rows[tid] = gather && r < n ? kv * L + idx[(size_t)h * L + r] : kv_rows;
        if (out.n) sm.drop[tid] = r < L && __ldg(inv + (size_t)h * L + r) < 0;
    }
    if (tid == 0 && gather) {
        mbar_init(&sm.full, 1);
        fence_barrier_init();
    }
    __syncthreads();
    if (gather && tid == 0) {
        const int nr = min(GT_ROWS, pad_end - r0);
        const int ng = (nr + 3) / 4;
        mbar_arrive_expect_tx(&sm.full, ng * 4 * 256 * 2);
        for (int g4 = 0; g4 < ng; ++g4) {
            const int* rr = sm.rows + 4 * g4;
            tma_gather4(sm.k + g4 * 1024, &tm_k, &sm.full, 0, rr[0], rr[1], rr[2], rr[3]);
            tma_gather4(sm.v + g4 * 1024, &tm_v, &sm.full, 0, rr[0], rr[1], rr[2], rr[3]);
        }
    }
    if (out.n) {  // zero rows of the dropped positions, every replica
#pragma unroll
        for (int i = 0; i < TSA_MAX_REPLICAS; ++i) {
            if (i >= out.n) break;
            uint4* o = static_cast<uint4*>(out.p[i]) + ((size_t)h * L + r0) * 16;
            for (int e = tid; e < GT_ROWS * 16; e += 256)
                if (sm.drop[e >> 4]) __stcs(o + e, make_uint4(0u, 0u, 0u, 0u));
        }
        if (out.n > 1) __threadfence_system();
    }
    if (gather && tid == 0) {
        mbar_wait(&sm.full, 0);
        fence_proxy_async_smem();
        // 64 rows per tensor in one store; the 3-D map clips rows >= L (never the
        // next head's); rows in (pad_end, r0 + 64) are scratch the attention skips
        tma_store_3d(&tm_kc, sm.k, 0, r0, h);
        tma_store_3d(&tm_vc, sm.v, 0, r0, h);
        bulk_commit();
        // only the shared-memory reads need to finish before the CTA ends (the writes
        // complete with the grid); waiting for them would hold the CTA's slot
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
}

template <typename V>
__global__ void __launch_bounds__(256) scatter_kernel(const V* __restrict__ oc,
                                                      const int32_t* __restrict__ inv,
                                                      V* __restrict__ out, int L, int chunks,
                                                      int head_begin) {
    const int h = head_begin + blockIdx.y;
    const int rows_per_block = 64;
    const int t0 = blockIdx.x * rows_per_block;
    const int32_t* inv_h = inv + (size_t)h * L;
    const int total = rows_per_block * chunks;
    for (int e = threadIdx.x; e < total; e += 256) {
        const int t = t0 + e / chunks, c = e % chunks;
        if (t >= L) break;
        const int r = inv_h[t];
        V val = V{};
        if (r >= 0) val = __ldg(oc + ((size_t)h * L + r) * chunks + c);
        out[((size_t)h * L + t) * chunks + c] = val;
    }
}

// Rows the selection dropped are +0.0 (scatter_rows zero-initialises its
// output, tensor_ops.cpp:107); the fused attention writes the kept rows.
template <typename V>
__global__ void __launch_bounds__(256) zero_unselected_kernel(const int32_t* __restrict__ inv,
                                                              V* __restrict__ out, int L,
                                                              int chunks, int head_begin) {
    const int h = head_begin + blockIdx.y;
    const int rows_per_block = 64;
    const int t0 = blockIdx.x * rows_per_block;
    const int32_t* inv_h = inv + (size_t)h * L;
    for (int e = threadIdx.x; e < rows_per_block * chunks; e += 256) {
        const int t = t0 + e / chunks, c = e % chunks;
        if (t >= L) break;
        if (inv_h[t] < 0) out[((size_t)h * L + t) * chunks + c] = V{};
    }
}

__global__ void inverse_fill_kernel(int32_t* __restrict__ inv, int L, int head_begin) {
    const int h = head_begin + blockIdx.y;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < L) inv[(size_t)h * L + t] = -1;
}

__global__ void inverse_set_kernel(const int32_t* __restrict__ idx, const int32_t* __restrict__ k_keep_p,
                                   int32_t* __restrict__ inv, int L, int head_begin) {
    const int h = head_begin + blockIdx.y;
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < *k_keep_p) inv[(size_t)h * L + idx[(size_t)h * L + r]] = r;
}

}  // namespace

// inv[h, t] = r where idx[h, r] == t, else -1 (for a caller-supplied selection).
int launch_inverse(const tsa_desc& d, const int32_t* idx, const int32_t* k_keep, int32_t* inv,
                   cudaStream_t st) {
    const int L = d.seq_len, nh = d.head_end - d.head_begin;
    dim3 grid((L + 255) / 256, nh);
    inverse_fill_kernel<<<grid, 256, 0, st>>>(inv, L, d.head_begin);
    inverse_set_kernel<<<grid, 256, 0, st>>>(idx, k_keep, inv, L, d.head_begin);
    TSA_LAUNCH_CHECK("inverse");
    return 0;
}

// Row access width: 16, 4 or 2 bytes.
static int unit_bytes(const tsa_desc& d) {
    const size_t row = d.d_head * elem_bytes(d.dtype);
    return row % 16 == 0 ? 16 : row % 4 == 0 ? 4 : 2;
}

template <typename V>
static int zero_t(const tsa_desc& d, const int32_t* inv, void* out, cudaStream_t st) {
    const int L = d.seq_len;
    const int chunks = (int)(d.d_head * elem_bytes(d.dtype) / sizeof(V));
    dim3 grid((L + 63) / 64, d.head_end - d.head_begin);
    zero_unselected_kernel<V><<<grid, 256, 0, st>>>(inv, (V*)out, L, chunks, d.head_begin);
    TSA_LAUNCH_CHECK("zero_unselected");
    return 0;
}

int launch_zero_unselected(const tsa_desc& d, const int32_t* inv, void* out, cudaStream_t st) {
    switch (unit_bytes(d)) {
        case 16: return zero_t<uint4>(d, inv, out, st);
        case 4: return zero_t<uint32_t>(d, inv, out, st);
        default: return zero_t<uint16_t>(d, inv, out, st);
    }
}

template <typename V>
static int gather_t(const tsa_desc& d, const void* q, const void* k, const void* v,
                    const int32_t* idx, const int32_t* k_keep, void* qc, void* kc, void* vc,
                    const int32_t* inv, const OutReplicas& out, cudaStream_t st) {
    const int L = d.seq_len;
    const int chunks = (int)(d.d_head * elem_bytes(d.dtype) / sizeof(V));
    const int nh = d.head_end - d.head_begin;
    const int group = d.n_heads / d.n_kv_heads;  // shards hold whole KV groups
    dim3 grid((L + 63) / 64 * group, nh / group);
    const int skip = (qc == nullptr && out.n > 0) ? 1 : 0;
    if (sizeof(V) == 16 && chunks == 16 && d.dtype == TSA_BF16 && qc == nullptr && skip) {
        // the fused path's K/V compress: TMA row gathers and bulk row stores
        const int kv_begin = d.head_begin / group, n_kv = nh / group;
        const uint8_t* kb = static_cast<const uint8_t*>(k) + (size_t)kv_begin * L * 256;
        const uint8_t* vb = static_cast<const uint8_t*>(v) + (size_t)kv_begin * L * 256;
        CUtensorMap mk, mv, mkc, mvc;
        int rc;
        if ((rc = make_bf16_rows_map(&mk, kb, (uint64_t)n_kv * L, 1)) ||
            (rc = make_bf16_rows_map(&mv, vb, (uint64_t)n_kv * L, 1)) ||
            (rc = make_bf16_rows_map_3d(&mkc, kc, L, d.head_end, GT_ROWS)) ||
            (rc = make_bf16_rows_map_3d(&mvc, vc, L, d.head_end, GT_ROWS)))
            return rc;
        gather_tma_kernel<<<grid, 256, 0, st>>>(mk, mv, mkc, mvc, idx, k_keep, L, group,
                                                 d.head_begin, n_kv * L, inv, out);
        TSA_LAUNCH_CHECK("gather_tma");
        return 0;
    }
    if (sizeof(V) == 16 && chunks == 16)  // d = 128 bf16 rows
        gather_kernel<V, 16><<<grid, 256, 0, st>>>((const V*)q, (const V*)k, (const V*)v, idx,
                                                   k_keep, (V*)qc, (V*)kc, (V*)vc, L, group,
                                                   chunks, d.head_begin, inv, out, skip);
    else
        gather_kernel<V, 0><<<grid, 256, 0, st>>>((const V*)q, (const V*)k, (const V*)v, idx,
                                                  k_keep, (V*)qc, (V*)kc, (V*)vc, L, group,
                                                  chunks, d.head_begin, inv, out, skip);
    TSA_LAUNCH_CHECK("gather");
    return 0;
}

static int gather_dispatch(const tsa_desc& d, const void* q, const void* k, const void* v,
                           const int32_t* idx, const int32_t* k_keep, void* qc, void* kc,
                           void* vc, const int32_t* inv, const OutReplicas& out,
                           cudaStream_t st) {
    switch (unit_bytes(d)) {
        case 16: return gather_t<uint4>(d, q, k, v, idx, k_keep, qc, kc, vc, inv, out, st);
        case 4: return gather_t<uint32_t>(d, q, k, v, idx, k_keep, qc, kc, vc, inv, out, st);
        default: return gather_t<uint16_t>(d, q, k, v, idx, k_keep, qc, kc, vc, inv, out, st);
    }
}

int launch_gather_zero(const tsa_desc& d, const void* q, const void* k, const void* v,
                       const int32_t* idx, const int32_t* k_keep, void* qc, void* kc, void* vc,
                       const int32_t* inv, void* out, cudaStream_t st) {
    OutReplicas r{};
    if (out) r = single_replica(out);
    return gather_dispatch(d, q, k, v, idx, k_keep, qc, kc, vc, inv, r, st);
}

int launch_gather_zero_rep(const tsa_desc& d, const void* k, const void* v, const int32_t* idx,
                           const int32_t* k_keep, void* kc, void* vc, const int32_t* inv,
                           const OutReplicas& out, cudaStream_t st) {
    return gather_dispatch(d, nullptr, k, v, idx, k_keep, nullptr, kc, vc, inv, out, st);
}

int launch_gather(const tsa_desc& d, const void* q, const void* k, const void* v,
                  const int32_t* idx, const int32_t* k_keep, void* qc, void* kc, void* vc,
                  cudaStream_t st) {
    return launch_gather_zero(d, q, k, v, idx, k_keep, qc, kc, vc, nullptr, nullptr, st);
}

template <typename V>
static int scatter_t(const tsa_desc& d, const void* oc, const int32_t* inv, void* out,
                     cudaStream_t st) {
    const int L = d.seq_len;
    const int chunks = (int)(d.d_head * elem_bytes(d.dtype) / sizeof(V));
    const int nh = d.head_end - d.head_begin;
    dim3 grid((L + 63) / 64, nh);
    scatter_kernel<V><<<grid, 256, 0, st>>>((const V*)oc, inv, (V*)out, L, chunks, d.head_begin);
    TSA_LAUNCH_CHECK("scatter");
    return 0;
}

int launch_scatter(const tsa_desc& d, const void* oc, const int32_t* inv, void* out,
                   cudaStream_t st) {
    switch (unit_bytes(d)) {
        case 16: return scatter_t<uint4>(d, oc, inv, out, st);
        case 4: return scatter_t<uint32_t>(d, oc, inv, out, st);
        default: return scatter_t<uint16_t>(d, oc, inv, out, st);
    }
}

}  // namespace tsa
