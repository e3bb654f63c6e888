// The reference's sequential f32 sum, bit for bit, without the sequential
// chain (select.cu: the budget's total, token_coverage.cpp:58-61;
// score_exact.cu: the row sums of softmax_rows, tensor_ops.cpp:59-65, when the
// rows are too few to hide their L-long chains).  See exact_chain_sum below.
#pragma once

#include <cooperative_groups.h>

#include <cstdint>

namespace tsa_dev {

// Block-wide exclusive scan of one double per thread; *total gets the sum.
template <int NT>
__device__ double chain_block_excl_scan(double v, double* total) {
    __shared__ double warp_sums[32];
    __shared__ double s_total;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double n = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += n;
    }
    if (lane == 31) warp_sums[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const double w = lane < NT / 32 ? warp_sums[lane] : 0.0;
        double wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double n = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += n;
        }
        if (lane < NT / 32) warp_sums[lane] = wi - w;
    }
    __syncthreads();
    const double excl = warp_sums[warp] + incl - v;
    if (threadIdx.x == NT - 1) s_total = excl + v;
    __syncthreads();
    *total = s_total;
    return excl;
}

// ------------------------------------------------- exact sequential f32 sum
// The reference's total (token_coverage.cpp:58-61): S_0 = +0, S_i = RN(S_{i-1}
// + x_i) over n non-negative floats, bit for bit, without n dependent adds.
// While S stays in one binade [2^E, 2^(E+1)) (ulp u = 2^(E-23), S = a u with
// integer a in [2^23, 2^24)), adding x = (k + f) u (k integer, f in [0,1),
// exact: scaling by a power of two) gives S' = (a + k + r) u with r = [f >
// 1/2] -- or, at an exact tie f = 1/2, the r that makes a + k + r even.  So a
// run of elements acts on S through its total increment, which depends on S
// only through E and the parity of a: per start parity the run is a pair
// (increment, end parity), and such pairs compose associatively (a monoid).
// Each thread folds one chunk under the binade its start probably has (from
// an approximate double prefix); warp 0 then walks the chunks in order with
// the exact S, 32 at a time: if every chunk of the group was folded under
// S's binade, a shuffle scan composes them and, when a + increment <= 2^24
// (no crossing inside: the partial sums are monotone), the group costs one
// step; otherwise its chunks are taken one at a time, and a chunk that
// crosses a power of two (or was folded under a wrong guess) is added element
// by element.  Exact by construction.
struct ChainFold {
    uint32_t inc0, inc1;  // total increment (units of u) for start parity 0 / 1
    uint32_t q0, q1;      // end parity for start parity 0 / 1
};

__device__ __forceinline__ ChainFold chain_compose(const ChainFold& f, const ChainFold& g) {
    ChainFold r;
    r.inc0 = f.inc0 + (f.q0 ? g.inc1 : g.inc0);
    r.q0 = f.q0 ? g.q1 : g.q0;
    r.inc1 = f.inc1 + (f.q1 ? g.inc1 : g.inc0);
    r.q1 = f.q1 ? g.q1 : g.q0;
    return r;
}

__device__ __forceinline__ void chain_fold_elem(ChainFold& m, float y) {
    const uint32_t k = (uint32_t)y;
    const float f = __fsub_rn(y, (float)k);
    const bool tie = f == 0.5f;
    const uint32_t r = f > 0.5f ? 1u : 0u;
    const uint32_t e0 = tie ? k + ((m.q0 + k) & 1u) : k + r;
    const uint32_t e1 = tie ? k + ((m.q1 + k) & 1u) : k + r;
    m.inc0 += e0;
    m.inc1 += e1;
    m.q0 = (m.q0 + e0) & 1u;
    m.q1 = (m.q1 + e1) & 1u;
}

// Chunks of CH = 256 * ceil(n / 128K) elements (at most kChainChunks), each
// folded by one warp with coalesced loads: lane l folds its CH/32 consecutive
// elements, a shuffle scan composes the lanes in order.
constexpr int kChainChunks = 512;

__device__ __forceinline__ ChainFold chain_warp_compose(ChainFold f, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        ChainFold p;
        p.inc0 = __shfl_up_sync(0xffffffffu, f.inc0, o);
        p.inc1 = __shfl_up_sync(0xffffffffu, f.inc1, o);
        p.q0 = __shfl_up_sync(0xffffffffu, f.q0, o);
        p.q1 = __shfl_up_sync(0xffffffffu, f.q1, o);
        if (lane >= o) f = chain_compose(p, f);
    }
    return f;  // lane 31: the whole warp's run
}

template <int NT>
__device__ float exact_chain_sum(const float* __restrict__ x, int n) {
    static_assert(NT % 32 == 0, "whole warps");
    constexpr int NW = NT / 32;
    constexpr int kChainStage = 256;
    __shared__ uint4 cm[kChainChunks];  // inc0, inc1, (E + 128) | q0 << 16 | q1 << 17, valid
    __shared__ double csum[kChainChunks];
    __shared__ float stage[kChainStage];
    __shared__ float s_res;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int CH = 256 * ((n + 256 * kChainChunks - 1) / (256 * kChainChunks));
    const int nch = (n + CH - 1) / CH;
    const int per = CH / 32;  // elements per lane: 8 (n <= 128K), a multiple of 8
    // phase 1: chunk sums (double) -> approximate exclusive prefix of each chunk
    // start; a warp takes 4 chunks per step so 8 x 16 B per lane are in flight
    const float4* x4 = reinterpret_cast<const float4*>(x);
    auto load8 = [&](int c, int q, float (&v)[8]) {  // lane's elements [q, q + 8) of chunk c
        const int b = c * CH + lane * per + q;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int i = b + 4 * h;
            float4 w = make_float4(0.f, 0.f, 0.f, 0.f);
            if (c < nch && i + 4 <= n) w = __ldg(x4 + i / 4);
            else if (c < nch)
                for (int j = 0; j < 4; ++j) (&w.x)[j] = i + j < n ? __ldg(x + i + j) : 0.0f;
            v[4 * h] = w.x, v[4 * h + 1] = w.y, v[4 * h + 2] = w.z, v[4 * h + 3] = w.w;
        }
    };
    for (int c0 = 4 * warp; c0 < nch; c0 += 4 * NW) {
        double ds4[4] = {0.0, 0.0, 0.0, 0.0};
        for (int q = 0; q < per; q += 8) {
            float v[4][8];
#pragma unroll
            for (int u = 0; u < 4; ++u) load8(c0 + u, q, v[u]);
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int j = 0; j < 8; ++j) ds4[u] += (double)v[u][j];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            double ds = ds4[u];
#pragma unroll
            for (int o = 16; o; o >>= 1) ds += __shfl_xor_sync(0xffffffffu, ds, o);
            if (lane == 0 && c0 + u < nch) csum[c0 + u] = ds;
        }
    }
    __syncthreads();
    {   // exclusive scan over the chunks, two per thread (nch <= 2 NT)
        const int c0 = 2 * t;
        const double a0 = c0 < nch ? csum[c0] : 0.0, a1 = c0 + 1 < nch ? csum[c0 + 1] : 0.0;
        double tot;
        const double ex = chain_block_excl_scan<NT>(a0 + a1, &tot);
        __syncthreads();
        if (c0 < nch) csum[c0] = ex;
        if (c0 + 1 < nch) csum[c0 + 1] = ex + a0;
    }
    __syncthreads();
    // phase 2: each chunk folded under the binade its start probably has
    for (int c0 = 4 * warp; c0 < nch; c0 += 4 * NW) {
        int E4[4];
        bool valid4[4];
        float scale4[4];
        ChainFold f4[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const float pf = c0 + u < nch ? (float)csum[c0 + u] : 0.0f;
            E4[u] = pf > 0.0f ? (int)((__float_as_uint(pf) >> 23) & 0xFF) - 127 : -1000;
            valid4[u] = E4[u] >= -100 && E4[u] <= 100;
            scale4[u] = valid4[u] ? __uint_as_float((uint32_t)(127 + 23 - E4[u]) << 23) : 1.0f;  // 2^(23-E)
            f4[u] = ChainFold{0u, 0u, 0u, 1u};
        }
        for (int q = 0; q < per; q += 8) {
            float v[4][8];
#pragma unroll
            for (int u = 0; u < 4; ++u) load8(c0 + u, q, v[u]);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const float y = __fmul_rn(v[u][j], scale4[u]);  // exact: power-of-two scaling
                    if (!(y < 16777216.0f)) valid4[u] = false;      // >= 2^24 u: crosses a binade
                    else chain_fold_elem(f4[u], y);
                }
                if (f4[u].inc0 > (1u << 25) || f4[u].inc1 > (1u << 25)) valid4[u] = false;
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int c = c0 + u;
            if (c >= nch) break;  // warp-uniform
            const int E = E4[u];
            bool valid = valid4[u];
            ChainFold f = f4[u];
            valid = __all_sync(0xffffffffu, valid);
            f = chain_warp_compose(f, lane);
            if (lane == 31)
                cm[c] = make_uint4(f.inc0, f.inc1, (uint32_t)(E + 128) | (f.q0 << 16) | (f.q1 << 17),
                                   (valid && f.inc0 <= (1u << 25) && f.inc1 <= (1u << 25)) ? 1u : 0u);
        }
    }
    __syncthreads();
    // phase 3: warp 0 walks the chunks with the exact running sum
    if (warp == 0) {
        float S = 0.0f;
        auto add_chunk = [&](int c) {  // one chunk, lane-uniform
            const int cb = c * CH, ce = min(n, cb + CH);
            const uint4 w = cm[c];
            const uint32_t bits = __float_as_uint(S);
            const int Es = (int)((bits >> 23) & 0xFF) - 127;
            if (w.w && (bits >> 23) != 0 && Es == (int)(w.z & 0xFFFFu) - 128) {
                const uint32_t a = (bits & 0x7FFFFFu) | 0x800000u;
                const uint32_t inc = (a & 1u) ? w.y : w.x;
                if (a + inc <= (1u << 24)) {
                    S = __fmul_rn((float)(a + inc), __uint_as_float((uint32_t)(127 + Es - 23) << 23));
                    return;
                }
            }
            // element by element: the warp stages the chunk in shared memory
            // (coalesced), then every lane runs the same f32 chain from it
            for (int sb = cb; sb < ce; sb += kChainStage) {
                const int m = min(kChainStage, ce - sb);
                for (int i = lane; i < m; i += 32) stage[i] = __ldg(x + sb + i);
                __syncwarp();
#pragma unroll 8
                for (int i = 0; i < m; ++i) S = __fadd_rn(S, stage[i]);
                __syncwarp();
            }
        };
        // 32 chunks per step: the leading run of chunks that were folded under
        // S's binade and keep a + increment <= 2^24 is applied at once; the
        // chunk after it (a crossing or a wrong guess) is added element by element
        int pos = 0;
        while (pos < nch) {
            const int c = pos + lane;
            const bool live = c < nch;
            const uint4 w = live ? cm[c] : make_uint4(0u, 0u, 0u, 0u);
            const uint32_t bits = __float_as_uint(S);
            const int Es = (int)((bits >> 23) & 0xFF) - 127;
            const bool normal = (bits >> 23) != 0;
            const bool folded = live && w.w && normal && Es == (int)(w.z & 0xFFFFu) - 128;
            ChainFold f = live ? ChainFold{w.x, w.y, (w.z >> 16) & 1u, (w.z >> 17) & 1u}
                               : ChainFold{0u, 0u, 0u, 1u};
            f = chain_warp_compose(f, lane);  // inclusive prefix (each chunk's inc <= 2^25)
            const uint32_t a = (bits & 0x7FFFFFu) | 0x800000u;
            const uint32_t inc = (a & 1u) ? f.inc1 : f.inc0;
            const bool good = folded && a + inc <= (1u << 24);
            const uint32_t ball = __ballot_sync(0xffffffffu, good);
            const int lead = ball == 0xffffffffu ? 32 : __ffs(~ball) - 1;
            if (lead > 0) {
                const uint32_t tot = __shfl_sync(0xffffffffu, inc, lead - 1);
                S = __fmul_rn((float)(a + tot), __uint_as_float((uint32_t)(127 + Es - 23) << 23));
            }
            pos += lead;
            if (lead < 32 && pos < nch) add_chunk(pos++);
        }
        if (lane == 0) s_res = S;
    }
    __syncthreads();
    return s_res;
}


// The same sum over a thread-block cluster of CLN CTAs whose slices of x
// ([r S, (r+1) S), S = ceil(n / CLN), in rank order) are staged in each CTA's
// shared memory (xs = this CTA's slice, ns its length, at most 64 chunks of
// 256): every CTA folds its own chunks, the chunk sums, their prefix and the
// folds meet in rank 0's shared memory through DSMEM, and rank 0's warp 0 walks
// them.  The result is returned in rank 0 (other ranks: undefined).
template <int NT, int CLN>
__device__ float cluster_exact_chain_sum(const float* xs, int ns, const float* __restrict__ x,
                                         int n) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    static_assert(NT % 32 == 0, "whole warps");
    constexpr int NW = NT / 32, CH = 256, PER = CH / 32;
    constexpr int kMaxChunks = kChainChunks;
    __shared__ uint4 cm[kMaxChunks];
    __shared__ double csum[kMaxChunks];
    __shared__ float stage[CH];
    __shared__ float s_res;
    const int rank = (int)cluster.block_rank();
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int S = (n + CLN - 1) / CLN;
    const int cpr = (S + CH - 1) / CH;  // chunks per rank (the last rank may have fewer)
    const int base = rank * cpr, nloc = (ns + CH - 1) / CH;
    const int last_len = n - (CLN - 1) * S;
    const int nch = (CLN - 1) * cpr + (last_len > 0 ? (last_len + CH - 1) / CH : 0);
    uint4* cm0 = cluster.map_shared_rank(cm, 0);
    double* csum0 = cluster.map_shared_rank(csum, 0);
    auto load8 = [&](int lc, float (&v)[PER]) {  // this lane's 8 elements of local chunk lc
        const int i0 = lc * CH + lane * PER;
#pragma unroll
        for (int j = 0; j < PER; ++j) v[j] = i0 + j < ns ? xs[i0 + j] : 0.0f;
    };
    cluster.sync();  // every CTA runs before any remote write
    // phase 1: chunk sums (double) into rank 0
    for (int lc = warp; lc < nloc; lc += NW) {
        float v[PER];
        load8(lc, v);
        double ds = 0.0;
#pragma unroll
        for (int j = 0; j < PER; ++j) ds += (double)v[j];
#pragma unroll
        for (int o = 16; o; o >>= 1) ds += __shfl_xor_sync(0xffffffffu, ds, o);
        if (lane == 0) csum0[base + lc] = ds;
    }
    cluster.sync();
    if (rank == 0) {  // exclusive prefix over the chunks, two per thread (nch <= 2 NT)
        const int c0 = 2 * t;
        const double a0 = c0 < nch ? csum[c0] : 0.0, a1 = c0 + 1 < nch ? csum[c0 + 1] : 0.0;
        double tot;
        const double ex = chain_block_excl_scan<NT>(a0 + a1, &tot);
        __syncthreads();
        if (c0 < nch) csum[c0] = ex;
        if (c0 + 1 < nch) csum[c0 + 1] = ex + a0;
    }
    cluster.sync();
    // phase 2: each chunk folded under the binade its start probably has
    for (int lc = warp; lc < nloc; lc += NW) {
        const float pf = (float)csum0[base + lc];
        const int E = pf > 0.0f ? (int)((__float_as_uint(pf) >> 23) & 0xFF) - 127 : -1000;
        bool valid = E >= -100 && E <= 100;
        ChainFold f{0u, 0u, 0u, 1u};
        if (valid) {
            const float scale = __uint_as_float((uint32_t)(127 + 23 - E) << 23);  // 2^(23 - E)
            float v[PER];
            load8(lc, v);
#pragma unroll
            for (int j = 0; j < PER; ++j) {
                const float y = __fmul_rn(v[j], scale);  // exact: power-of-two scaling
                if (!(y < 16777216.0f)) valid = false;   // >= 2^24 u: crosses a binade
                else chain_fold_elem(f, y);
            }
            if (f.inc0 > (1u << 25) || f.inc1 > (1u << 25)) valid = false;
        }
        valid = __all_sync(0xffffffffu, valid);
        f = chain_warp_compose(f, lane);
        if (lane == 31)
            cm0[base + lc] = make_uint4(f.inc0, f.inc1, (uint32_t)(E + 128) | (f.q0 << 16) | (f.q1 << 17),
                                        (valid && f.inc0 <= (1u << 25) && f.inc1 <= (1u << 25)) ? 1u : 0u);
    }
    cluster.sync();
    // phase 3: rank 0's warp 0 walks the chunks with the exact running sum
    if (rank == 0 && warp == 0) {
        float S_ = 0.0f;
        auto range = [&](int c, int& cb, int& ce) {
            const int r = c / cpr, lc = c % cpr;
            cb = r * S + lc * CH;
            ce = min(min(n, (r + 1) * S), cb + CH);
        };
        auto add_chunk = [&](int c) {  // one chunk, lane-uniform
            int cb, ce;
            range(c, cb, ce);
            const uint4 w = cm[c];
            const uint32_t bits = __float_as_uint(S_);
            const int Es = (int)((bits >> 23) & 0xFF) - 127;
            if (w.w && (bits >> 23) != 0 && Es == (int)(w.z & 0xFFFFu) - 128) {
                const uint32_t a = (bits & 0x7FFFFFu) | 0x800000u;
                const uint32_t inc = (a & 1u) ? w.y : w.x;
                if (a + inc <= (1u << 24)) {
                    S_ = __fmul_rn((float)(a + inc), __uint_as_float((uint32_t)(127 + Es - 23) << 23));
                    return;
                }
            }
            const int m = ce - cb;  // element by element, staged (coalesced)
            for (int i = lane; i < m; i += 32) stage[i] = __ldg(x + cb + i);
            __syncwarp();
#pragma unroll 8
            for (int i = 0; i < m; ++i) S_ = __fadd_rn(S_, stage[i]);
            __syncwarp();
        };
        int pos = 0;
        while (pos < nch) {
            const int c = pos + lane;
            const bool live = c < nch;
            const uint4 w = live ? cm[c] : make_uint4(0u, 0u, 0u, 0u);
            const uint32_t bits = __float_as_uint(S_);
            const int Es = (int)((bits >> 23) & 0xFF) - 127;
            const bool normal = (bits >> 23) != 0;
            const bool folded = live && w.w && normal && Es == (int)(w.z & 0xFFFFu) - 128;
            ChainFold f = live ? ChainFold{w.x, w.y, (w.z >> 16) & 1u, (w.z >> 17) & 1u}
                               : ChainFold{0u, 0u, 0u, 1u};
            f = chain_warp_compose(f, lane);
            const uint32_t a = (bits & 0x7FFFFFu) | 0x800000u;
            const uint32_t inc = (a & 1u) ? f.inc1 : f.inc0;
            const bool good = folded && a + inc <= (1u << 24);
            const uint32_t ball = __ballot_sync(0xffffffffu, good);
            const int lead = ball == 0xffffffffu ? 32 : __ffs(~ball) - 1;
            if (lead > 0) {
                const uint32_t tot = __shfl_sync(0xffffffffu, inc, lead - 1);
                S_ = __fmul_rn((float)(a + tot), __uint_as_float((uint32_t)(127 + Es - 23) << 23));
            }
            pos += lead;
            if (lead < 32 && pos < nch) add_chunk(pos++);
        }
        if (lane == 0) s_res = S_;
    }
    __syncthreads();
    return s_res;
}


// One warp's exact sequential f32 sum of x[0..n) (all lanes get it), streaming:
// per round each lane takes a chunk of 32 consecutive elements, a warp scan of
// the chunk sums (double) predicts each chunk's binade, each lane folds its
// chunk, and the exact running sum walks the round's chunks (leading run at
// once; the chunk after it element by element).  For rows of a few thousand
// elements (the REFERENCE-order softmax, tensor_ops.cpp:59-65).
__device__ __forceinline__ float warp_exact_chain_sum(const float* __restrict__ x, int n) {
    const int lane = threadIdx.x & 31;
    float S = 0.0f;
    double approx = 0.0;
    for (int base = 0; base < n; base += 32 * 32) {
        const int c0 = base + lane * 32;
        const int cnt = max(0, min(32, n - c0));
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = i < cnt ? x[c0 + i] : 0.0f;
        double ds = 0.0;
#pragma unroll
        for (int i = 0; i < 32; ++i) ds += (double)v[i];
        double incl = ds;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        const float pf = (float)(approx + incl - ds);
        approx += __shfl_sync(0xffffffffu, incl, 31);
        const int E = pf > 0.0f ? (int)((__float_as_uint(pf) >> 23) & 0xFF) - 127 : -1000;
        bool valid = cnt > 0 && E >= -100 && E <= 100;
        ChainFold f{0u, 0u, 0u, 1u};
        if (valid) {
            const float scale = __uint_as_float((uint32_t)(127 + 23 - E) << 23);  // 2^(23 - E)
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                if (i < cnt) {
                    const float y = __fmul_rn(v[i], scale);
                    if (!(y < 16777216.0f)) valid = false;
                    else chain_fold_elem(f, y);
                }
            }
            if (f.inc0 > (1u << 25) || f.inc1 > (1u << 25)) valid = false;
        }
        int pos = 0;
        while (pos < 32) {
            const int cnt_pos = __shfl_sync(0xffffffffu, cnt, pos);
            if (cnt_pos == 0) break;  // past n
            const uint32_t bits = __float_as_uint(S);
            const int Es = (int)((bits >> 23) & 0xFF) - 127;
            const bool live = lane >= pos && cnt > 0;
            const bool folded = live && valid && (bits >> 23) != 0 && Es == E;
            ChainFold g = (lane >= pos) ? f : ChainFold{0u, 0u, 0u, 1u};
            g = chain_warp_compose(g, lane);
            const uint32_t a = (bits & 0x7FFFFFu) | 0x800000u;
            const uint32_t inc = (a & 1u) ? g.inc1 : g.inc0;
            const bool good = lane < pos || (folded && a + inc <= (1u << 24));
            const uint32_t ball = __ballot_sync(0xffffffffu, good);
            const int lead = ball == 0xffffffffu ? 32 : __ffs(~ball) - 1;
            if (lead > pos) {
                const uint32_t tot = __shfl_sync(0xffffffffu, inc, lead - 1);
                S = __fmul_rn((float)(a + tot), __uint_as_float((uint32_t)(127 + Es - 23) << 23));
            }
            pos = lead;
            if (pos < 32) {  // this chunk element by element (its values from lane pos)
                const int m = __shfl_sync(0xffffffffu, cnt, pos);
                float w[32];
#pragma unroll
                for (int i = 0; i < 32; ++i) w[i] = __shfl_sync(0xffffffffu, v[i], pos);
#pragma unroll
                for (int i = 0; i < 32; ++i)
                    if (i < m) S = __fadd_rn(S, w[i]);
                ++pos;
            }
        }
    }
    return S;
}

}  // namespace tsa_dev
