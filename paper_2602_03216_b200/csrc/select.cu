// K2 budget + K3 head-wise top-k selection.
//
// K2 (aggregate_scores + coverage_budget, token_coverage.cpp:52-96):
//   headsum[t] = sum_h s[h, t]          f32, h ascending (:55-57)  -- parallel over t
//   total      = sum_t headsum[t]       f32, t ascending (:58-61)  -- one sequential chain
//   s_l[t]     = headsum[t] / total     (:65)
//   k_sparse   = smallest k whose ascending prefix of s_l reaches tau (:78-94)
// The crossing is found by a 3-level radix select over the f32 bit patterns of
// s_l (ascending bit order == ascending value order for non-negative floats)
// with exact 2^-62 fixed-point masses, so the ascending order and its tie
// handling never have to be materialised: only the sorted *values* decide
// k_sparse, and tied values contribute identical masses.  The reference sums
// the prefix in double; the exact fixed-point sum differs from it by less than
// L * 2^-53, documented as the near-tie rule in DESIGN.md.
//
// Both run as thread-block clusters of 8 CTAs (the token axis split 8 ways,
// histograms merged through distributed shared memory).
// K3 (select_tokens, token_coverage.cpp:111-152), one cluster per head:
//   radix select of the (k - |F|)-th largest non-forced score, then one
//   ordered compaction pass: keep t if forced, if s > v*, or if s == v* and t
//   is among the lowest-index (k - |F| - count(> v*)) ties.  Output is
//   ascending by construction; the inverse map is written in the same pass.
#include <cooperative_groups.h>

#include "common.cuh"
#include "chain_sum.cuh"

namespace tsa {
namespace {

constexpr int BT = 1024;  // threads per budget/select CTA

__global__ void write_int_kernel(int32_t* dst, int32_t v) { *dst = v; }

// headsum[t] = sum over ALL heads (h ascending), f32.
__global__ void headsum_kernel(const float* __restrict__ s, float* __restrict__ out, int H, int L) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= L) return;
    float acc = 0.0f;
    for (int h = 0; h < H; ++h) acc = __fadd_rn(acc, s[(size_t)h * L + t]);
    out[t] = acc;
}

__device__ __forceinline__ uint32_t score_key(float x) {
    // scores are >= +0; fold -0 onto +0 so bit order == value order
    const uint32_t u = __float_as_uint(x);
    return (u == 0x80000000u) ? 0u : u;
}

// Levels of the 32-bit radix select: bits [21,32), [10,21), [0,10).
__device__ __constant__ int kShift[3] = {21, 10, 0};
__device__ __constant__ int kBits[3] = {11, 11, 10};

// Block-wide exclusive scan of `v` (one value per thread) -> returns exclusive
// prefix and writes the block total to *total (all threads).
template <typename U, int NT = BT>
__device__ U block_excl_scan(U v, U* total) {
    __shared__ U warp_sums[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    U incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const U n = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += n;
    }
    if (lane == 31) warp_sums[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        U w = lane < NT / 32 ? warp_sums[lane] : U(0);
        U wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const U n = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += n;
        }
        if (lane < NT / 32) warp_sums[lane] = wi - w;  // exclusive prefix of warp totals
    }
    __syncthreads();
    const U excl = warp_sums[warp] + incl - v;
    // total = exclusive prefix of the last warp + its inclusive sum
    __shared__ U s_total;
    if (threadIdx.x == NT - 1) s_total = excl + v;
    __syncthreads();
    *total = s_total;
    return excl;
}

// ---------------------------------------------------------------- budget
// Single CTA.  mode 1 = dynamic; fixed/dense k_keep values are written by the host.
// mode BUDGET_FROM_HEADSUM: s_l = headsum / total (total = sequential chain);
// mode BUDGET_FROM_SL:       values already are s_l (LayerScores input), total = 1;
// mode AGGREGATE_ONLY:       write s_l = headsum / total to sl_out and stop.
enum { BUDGET_FROM_HEADSUM = 0, BUDGET_FROM_SL = 1, AGGREGATE_ONLY = 2 };

constexpr int BB = 512;  // threads per budget CTA
constexpr int CL = 8;  // CTAs per cluster: the token axis of one head (or of s_l) is split 8 ways

// Sum of `v` over the block (all threads get it).
template <typename U, int NT = BT>
__device__ U block_sum(U v) {
    U tot;
    block_excl_scan<U, NT>(v, &tot);
    return tot;
}

// ---------------------------------------------------------------- budget
// One cluster of CL CTAs; CTA r owns tokens [r*S, (r+1)*S).  Per radix level:
// local warp-aggregated histograms (count + exact 2^-62 fixed-point mass),
// cluster barrier, CTA r merges bucket range r across the cluster through
// DSMEM, range totals decide which CTA holds the crossing, that CTA finds the
// bucket and broadcasts it into every CTA's shared memory.
template <bool kStaged>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(BB, 1)
budget_kernel(const float* __restrict__ headsum, int L, double tau, int min_keep,
              int32_t* __restrict__ k_keep, int32_t* __restrict__ status, int mode,
              float* __restrict__ sl_out, int exact_total) {
    // kStaged: this CTA's slice of headsum (then s_l) lives in shared memory,
    // so the three histogram levels do not re-read global memory; the four
    // 16-bit mass-limb histograms follow it
    extern __shared__ float staged[];
    uint32_t(*hist_limb)[2048] = reinterpret_cast<uint32_t(*)[2048]>(
        staged + ((L + CL - 1) / CL + 3) / 4 * 4);
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = (int)cluster.block_rank();
    const int tid = threadIdx.x;
    __shared__ uint32_t hist_cnt[2048];
    __shared__ unsigned long long hist_mass[2048];
    __shared__ uint32_t m_cnt[2048 / CL];
    __shared__ unsigned long long m_mass[2048 / CL];
    __shared__ uint32_t range_cnt;
    __shared__ unsigned long long range_mass;
    __shared__ double part_total;
    __shared__ float s_total;
    __shared__ uint32_t res_bucket, res_cnt;
    __shared__ unsigned long long res_mass;
    __shared__ int s_rstar;
    __shared__ unsigned long long s_below_r;
    __shared__ uint32_t s_cbelow_r;
    const int S = (L + CL - 1) / CL;
    const int t_begin = min(L, rank * S), t_end = min(L, t_begin + S);

    // ---- total ----
    float total = 1.0f;
    if (mode != BUDGET_FROM_SL) {
        if (exact_total) {
            // the sequential f32 chain (token_coverage.cpp:58-61), bit for bit:
            // staged slices -> the chunk folds spread over the cluster, walked in rank 0
            if (kStaged) {
                for (int t = t_begin + tid; t < t_end; t += BB) staged[t - t_begin] = headsum[t];
                __syncthreads();
                const float acc = tsa_dev::cluster_exact_chain_sum<BB, CL>(staged, t_end - t_begin,
                                                                          headsum, L);
                if (rank == 0 && tid == 0) s_total = acc;
            } else if (rank == 0) {
                const float acc = tsa_dev::exact_chain_sum<BB>(headsum, L);
                if (tid == 0) s_total = acc;
            }
            // (rank 0 publishes locally; the others read it through DSMEM after the
            // barrier -- no remote write may precede the first cluster barrier,
            // when a peer CTA may not have started yet)
            cluster.sync();
            total = *cluster.map_shared_rank(&s_total, 0);
        } else {
            // deterministic parallel f64 reduction (FAST scoring mode): fixed
            // per-CTA partials combined in rank order by every CTA
            double acc = 0.0;
            for (int t = t_begin + tid; t < t_end; t += BB) {
                const float x = headsum[t];
                acc += (double)x;
                if (kStaged) staged[t - t_begin] = x;
            }
            acc = block_sum<double, BB>(acc);
            if (tid == 0) part_total = acc;
            cluster.sync();
            double tot = 0.0;
            for (int r = 0; r < CL; ++r) tot += *cluster.map_shared_rank(&part_total, r);
            total = (float)tot;
        }
        if (!(total > 0.0f)) {  // aggregate_scores throws (:62-64)
            if (rank == 0 && tid == 0) {
                *status = 1;
                if (k_keep) *k_keep = min_keep;
            }
            cluster.sync();
            return;
        }
        if (mode == AGGREGATE_ONLY) {
            for (int t = t_begin + tid; t < t_end; t += BB) sl_out[t] = __fdiv_rn(headsum[t], total);
            cluster.sync();
            return;
        }
        if (kStaged)  // s_l = headsum / total in place (token_coverage.cpp:65)
            for (int i = tid; i < t_end - t_begin; i += BB) staged[i] = __fdiv_rn(staged[i], total);
    } else if (kStaged) {
        for (int t = t_begin + tid; t < t_end; t += BB) staged[t - t_begin] = headsum[t];
    }
    __syncthreads();
    // ---- coverage crossing ----
    // T = ceil(tau * 2^62); tau = 0 -> k_sparse = 0 (prefix 0 >= 0, :82).
    const double tscaled = ldexp(tau, 62);
    unsigned long long T = (unsigned long long)tscaled;
    if ((double)T < tscaled) ++T;
    if (T == 0ull) {
        if (rank == 0 && tid == 0) *k_keep = max(L, min_keep);
        cluster.sync();
        return;
    }
    uint32_t prefix = 0, cnt_below = 0;
    unsigned long long mass_below = 0;
    bool done = false;  // total mass never reaches tau: k_sparse = L
    for (int lvl = 0; lvl < 3; ++lvl) {
        const int shift = kShift[lvl], bits = kBits[lvl], nb = 1 << bits, per = nb / CL;
        const int pshift = shift + bits;
        for (int b = tid; b < nb; b += BB) {
            hist_cnt[b] = 0;
            hist_mass[b] = 0;
            if (kStaged)
                for (int l = 0; l < 4; ++l) hist_limb[l][b] = 0;
        }
        __syncthreads();
        for (int base = t_begin; base < t_end; base += BB) {
            const int t = base + tid;
            uint32_t b = 0xFFFFFFFFu;
            unsigned long long m = 0;
            if (t < t_end) {
                const float sl = kStaged ? staged[t - t_begin] : __fdiv_rn(headsum[t], total);
                const uint32_t key = score_key(sl);
                if (pshift >= 32 || (key >> pshift) == prefix) {
                    b = (key >> shift) & (nb - 1);
                    m = (unsigned long long)ldexp((double)sl, 62);
                }
            }
            if (kStaged) {
                // native 32-bit shared atomics per lane: the count and the mass in
                // four 16-bit limbs (a slice has <= 16384 tokens, so a limb sum
                // stays below 2^30); the group reductions of the general path
                // serialise over the distinct buckets of a warp
                if (b != 0xFFFFFFFFu) {
                    atomicAdd(&hist_cnt[b], 1u);
#pragma unroll
                    for (int l = 0; l < 4; ++l)
                        atomicAdd(&hist_limb[l][b], (uint32_t)((m >> (16 * l)) & 0xFFFFu));
                }
            } else {
                // lanes of one bucket combine count and mass (three 21-bit limbs so
                // the 32-lane sums cannot overflow) before one shared atomic
                const uint32_t grp = __match_any_sync(0xffffffffu, b);
                const uint32_t l0 = __reduce_add_sync(grp, (uint32_t)(m & 0x1FFFFFu));
                const uint32_t l1 = __reduce_add_sync(grp, (uint32_t)((m >> 21) & 0x1FFFFFu));
                const uint32_t l2 = __reduce_add_sync(grp, (uint32_t)(m >> 42));
                if (b != 0xFFFFFFFFu && (__ffs(grp) - 1) == (tid & 31)) {
                    atomicAdd(&hist_cnt[b], (uint32_t)__popc(grp));
                    atomicAdd(&hist_mass[b], (unsigned long long)l0 +
                                                 ((unsigned long long)l1 << 21) +
                                                 ((unsigned long long)l2 << 42));
                }
            }
        }
        if (kStaged) {
            __syncthreads();
            for (int b = tid; b < nb; b += BB)
                hist_mass[b] = (unsigned long long)hist_limb[0][b] +
                               ((unsigned long long)hist_limb[1][b] << 16) +
                               ((unsigned long long)hist_limb[2][b] << 32) +
                               ((unsigned long long)hist_limb[3][b] << 48);
        }
        cluster.sync();
        // merge bucket range [rank*per, (rank+1)*per) over the cluster
        uint32_t mc = 0;
        unsigned long long mm = 0;
        if (tid < per) {
            const int b = rank * per + tid;
            for (int r = 0; r < CL; ++r) {
                mc += cluster.map_shared_rank(hist_cnt, r)[b];
                mm += cluster.map_shared_rank(hist_mass, r)[b];
            }
            m_cnt[tid] = mc;
            m_mass[tid] = mm;
        }
        const uint32_t rc = block_sum<uint32_t, BB>(mc);
        const unsigned long long rmass = block_sum<unsigned long long, BB>(mm);
        if (tid == 0) {
            range_cnt = rc;
            range_mass = rmass;
        }
        cluster.sync();
        const unsigned long long need = T - mass_below;  // > 0
        if (tid == 0) {
            unsigned long long below = 0;
            uint32_t cbelow = 0;
            int rstar = -1;
            for (int r = 0; r < CL; ++r) {
                const unsigned long long mr = *cluster.map_shared_rank(&range_mass, r);
                const uint32_t cr = *cluster.map_shared_rank(&range_cnt, r);
                if (below < need && need <= below + mr) {
                    rstar = r;
                    break;
                }
                below += mr;
                cbelow += cr;
            }
            s_rstar = rstar;
            s_below_r = below;
            s_cbelow_r = cbelow;
        }
        __syncthreads();
        if (s_rstar < 0) {  // only possible at level 0: total mass < tau
            done = true;
            cluster.sync();
            break;
        }
        if (rank == s_rstar) {
            // ascending exclusive scan inside this CTA's merged range
            const unsigned long long m0 = tid < per ? m_mass[tid] : 0;
            const uint32_t c0 = tid < per ? m_cnt[tid] : 0;
            unsigned long long mtot;
            uint32_t ctot;
            const unsigned long long mex = block_excl_scan<unsigned long long, BB>(m0, &mtot) + s_below_r;
            const uint32_t cex = block_excl_scan<uint32_t, BB>(c0, &ctot) + s_cbelow_r;
            if (tid < per && mex < need && need <= mex + m0) {
                for (int r = 0; r < CL; ++r) {
                    *cluster.map_shared_rank(&res_bucket, r) = (uint32_t)(rank * per + tid);
                    *cluster.map_shared_rank(&res_mass, r) = mex;
                    *cluster.map_shared_rank(&res_cnt, r) = cex;
                }
            }
        }
        cluster.sync();
        prefix = (prefix << bits) | res_bucket;
        mass_below += res_mass;
        cnt_below += res_cnt;
        cluster.sync();  // everyone read res before the next level may overwrite it
    }
    if (rank == 0 && tid == 0) {
        int k_sparse = L;
        if (!done) {
            const float v = __uint_as_float(prefix);
            const unsigned long long m = (unsigned long long)ldexp((double)v, 62);
            const unsigned long long need = T - mass_below;
            const unsigned long long c = (need + m - 1) / m;  // m > 0: bucket mass crossed
            k_sparse = (int)(cnt_below + c);
        }
        *k_keep = max(L - k_sparse, min_keep);
    }
}

// ---------------------------------------------------------------- select
__device__ __forceinline__ bool is_forced(int t, const int32_t* forced, int nf, int fbegin) {
    if (fbegin >= 0) return t >= fbegin;  // contiguous suffix (both SparsePlan policies)
    int lo = 0, hi = nf;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (forced[mid] < t) lo = mid + 1;
        else hi = mid;
    }
    return lo < nf && forced[lo] == t;
}

// One cluster of CL CTAs per head; CTA r owns tokens [r*S, (r+1)*S).  Radix
// select of the (k - |F|)-th largest non-forced key as in budget_kernel
// (descending), then an ordered compaction whose per-slice bases (kept count
// and tie count before the slice) come from the lower-ranked CTAs via DSMEM.
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(BT, 1)
select_kernel(const float* __restrict__ s, int L, const int32_t* __restrict__ k_keep_p,
              const int32_t* __restrict__ forced, int nf, int fbegin, int head_begin,
              int32_t* __restrict__ idx, int32_t* __restrict__ inv) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = (int)cluster.block_rank();
    const int tid = threadIdx.x;
    __shared__ uint32_t hist[2048];
    __shared__ uint32_t m_cnt[2048 / CL];
    __shared__ uint32_t range_cnt;
    __shared__ uint32_t res_bucket, res_above;
    __shared__ int s_rstar;
    __shared__ uint32_t s_above_r;
    __shared__ int slice_fg, slice_eq;  // forced-or-greater and tie counts of this slice
    const int h = head_begin + blockIdx.y;
    const float* sh = s + (size_t)h * L;
    const int S = (L + CL - 1) / CL;
    const int t_begin = min(L, rank * S), t_end = min(L, t_begin + S);
    const int k_keep = *k_keep_p;
    const int n_free = k_keep - nf;
    uint32_t prefix = 0, need = (uint32_t)max(n_free, 0);
    if (n_free > 0) {
        for (int lvl = 0; lvl < 3; ++lvl) {
            const int shift = kShift[lvl], bits = kBits[lvl], nb = 1 << bits, per = nb / CL;
            const int pshift = shift + bits;
            for (int b = tid; b < nb; b += BT) hist[b] = 0;
            __syncthreads();
            for (int base = t_begin; base < t_end; base += BT) {
                const int t = base + tid;
                uint32_t b = 0xFFFFFFFFu;
                if (t < t_end && !is_forced(t, forced, nf, fbegin)) {
                    const uint32_t key = score_key(sh[t]);
                    if (pshift >= 32 || (key >> pshift) == prefix) b = (key >> shift) & (nb - 1);
                }
                const uint32_t grp = __match_any_sync(0xffffffffu, b);  // warp-aggregated
                if (b != 0xFFFFFFFFu && (__ffs(grp) - 1) == (tid & 31))
                    atomicAdd(&hist[b], (uint32_t)__popc(grp));
            }
            cluster.sync();
            uint32_t mc = 0;
            if (tid < per) {
                const int b = rank * per + tid;
                for (int r = 0; r < CL; ++r) mc += cluster.map_shared_rank(hist, r)[b];
                m_cnt[tid] = mc;
            }
            const uint32_t rc = block_sum<uint32_t>(mc);
            if (tid == 0) range_cnt = rc;
            cluster.sync();
            if (tid == 0) {  // descending over ranks: higher ranks hold higher buckets
                uint32_t above = 0;
                int rstar = -1;
                for (int r = CL - 1; r >= 0; --r) {
                    const uint32_t cr = *cluster.map_shared_rank(&range_cnt, r);
                    if (above < need && need <= above + cr) {
                        rstar = r;
                        break;
                    }
                    above += cr;
                }
                s_rstar = rstar;
                s_above_r = above;
            }
            __syncthreads();
            if (rank == s_rstar) {
                // descending exclusive scan: thread i handles bucket per-1-i
                const int bi = per - 1 - tid;
                const uint32_t c0 = (tid < per) ? m_cnt[bi] : 0;
                uint32_t ctot;
                const uint32_t above = block_excl_scan<uint32_t>(c0, &ctot) + s_above_r;
                if (tid < per && above < need && need <= above + c0) {
                    for (int r = 0; r < CL; ++r) {
                        *cluster.map_shared_rank(&res_bucket, r) = (uint32_t)(rank * per + bi);
                        *cluster.map_shared_rank(&res_above, r) = above;
                    }
                }
            }
            cluster.sync();
            prefix = (prefix << bits) | res_bucket;
            need -= res_above;
            cluster.sync();  // everyone read res before the next level may overwrite it
        }
    }
    const uint32_t vstar = prefix;
    const bool has_thr = n_free > 0;
    const int take_eq = has_thr ? (int)need : 0;  // ties at v* to keep, lowest index first
    // ---- slice counts -> bases from the lower-ranked CTAs ----
    int fg = 0, eq = 0;
    for (int t = t_begin + tid; t < t_end; t += BT) {
        const bool f = is_forced(t, forced, nf, fbegin);
        const uint32_t key = score_key(sh[t]);
        if (f || (has_thr && key > vstar)) ++fg;
        else if (has_thr && key == vstar) ++eq;
    }
    fg = block_sum<int>(fg);
    eq = block_sum<int>(eq);
    if (tid == 0) {
        slice_fg = fg;
        slice_eq = eq;
    }
    cluster.sync();
    int base_pos = 0, base_eq = 0;
    for (int r = 0; r < rank; ++r) {
        const int fr = *cluster.map_shared_rank(&slice_fg, r);
        const int er = *cluster.map_shared_rank(&slice_eq, r);
        base_pos += fr + max(0, min(er, take_eq - base_eq));
        base_eq += er;
    }
    cluster.sync();  // remote reads done before any CTA may exit
    // ---- ordered compaction of this slice ----
    int32_t* idx_h = idx + (size_t)h * L;
    int32_t* inv_h = inv ? inv + (size_t)h * L : nullptr;
    constexpr int IPT = 4;
    for (int t0 = t_begin; t0 < t_end; t0 += BT * IPT) {
        int keep_flags = 0, eq_flags = 0, nkeep = 0, neq = 0;
        uint32_t keys[IPT];
        bool forced_f[IPT];
#pragma unroll
        for (int i = 0; i < IPT; ++i) {
            const int t = t0 + tid * IPT + i;
            forced_f[i] = false;
            keys[i] = 0;
            if (t < t_end) {
                forced_f[i] = is_forced(t, forced, nf, fbegin);
                keys[i] = score_key(sh[t]);
                if (!forced_f[i] && has_thr && keys[i] == vstar) {
                    eq_flags |= 1 << i;
                    ++neq;
                }
            }
        }
        int eq_total;
        const int eq_before = block_excl_scan<int>(neq, &eq_total) + base_eq;
        int running_eq = eq_before;
#pragma unroll
        for (int i = 0; i < IPT; ++i) {
            const int t = t0 + tid * IPT + i;
            if (t >= t_end) continue;
            bool keep = forced_f[i];
            if (!keep && has_thr) {
                if (keys[i] > vstar) keep = true;
                else if (eq_flags & (1 << i)) keep = running_eq++ < take_eq;
            }
            if (keep) {
                keep_flags |= 1 << i;
                ++nkeep;
            }
        }
        int keep_total;
        int pos = block_excl_scan<int>(nkeep, &keep_total) + base_pos;
#pragma unroll
        for (int i = 0; i < IPT; ++i) {
            const int t = t0 + tid * IPT + i;
            if (t >= t_end) continue;
            if (keep_flags & (1 << i)) {
                idx_h[pos] = t;
                if (inv_h) inv_h[t] = pos;
                ++pos;
            } else if (inv_h) {
                inv_h[t] = -1;
            }
        }
        base_pos += keep_total;
        base_eq += eq_total;
    }
}

// ------------------------------------------------ select, slice in shared memory
// Same algorithm as select_kernel, with each CTA's slice of the head's scores
// staged once into shared memory as radix keys (forced tokens as the
// kForcedKey sentinel): the three histogram levels and the two compaction
// passes then read shared memory instead of re-reading L2 five times, and 384
// threads per CTA let two clusters share an SM without register spills.  Used when a slice fits
// (ceil(L / CL) <= kSliceMax).
constexpr int BS = 384;  // 2 CTAs per SM at <= 85 registers: no spills (512 spilled 56 B)
constexpr int kSliceMax = 16384;
constexpr uint32_t kForcedKey = 0xFFFFFFFFu;

__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(BS, 2)
select_smem_kernel(const float* __restrict__ s, int L, const int32_t* __restrict__ k_keep_p,
                   const int32_t* __restrict__ forced, int nf, int fbegin, int head_begin,
                   int32_t* __restrict__ idx, int32_t* __restrict__ inv) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ uint32_t keys[];  // this CTA's slice
    const int rank = (int)cluster.block_rank();
    const int tid = threadIdx.x;
    __shared__ uint32_t hist[2048];
    __shared__ uint32_t m_cnt[2048 / CL];
    __shared__ uint32_t range_cnt;
    __shared__ uint32_t res_bucket, res_above;
    __shared__ int s_rstar;
    __shared__ uint32_t s_above_r;
    __shared__ int slice_fg, slice_eq;
    const int h = head_begin + blockIdx.y;
    const float* sh = s + (size_t)h * L;
    const int S = (L + CL - 1) / CL;
    const int t_begin = min(L, rank * S), t_end = min(L, t_begin + S);
    const int n_loc = t_end - t_begin;
    const int k_keep = *k_keep_p;
    const int n_free = k_keep - nf;
    // ---- stage keys (8 independent loads in flight per thread) ----
    for (int i0 = 0; i0 < n_loc; i0 += BS * 8) {
        float v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = i0 + u * BS + tid;
            v[u] = i < n_loc ? __ldg(sh + t_begin + i) : 0.0f;
        }
#pragma unroll 4
        for (int u = 0; u < 8; ++u) {
            const int i = i0 + u * BS + tid;
            if (i < n_loc)
                keys[i] = is_forced(t_begin + i, forced, nf, fbegin) ? kForcedKey : score_key(v[u]);
        }
    }
    __syncthreads();
    uint32_t prefix = 0, need = (uint32_t)max(n_free, 0);
    if (n_free > 0) {
        for (int lvl = 0; lvl < 3; ++lvl) {
            const int shift = kShift[lvl], bits = kBits[lvl], nb = 1 << bits, per = nb / CL;
            const int pshift = shift + bits;
            for (int b = tid; b < nb; b += BS) hist[b] = 0;
            __syncthreads();
            for (int i0 = 0; i0 < n_loc; i0 += BS) {  // whole warps iterate together
                const int i = i0 + tid;
                const uint32_t key = i < n_loc ? keys[i] : kForcedKey;
                uint32_t b = 0xFFFFFFFFu;
                if (key != kForcedKey && (pshift >= 32 || (key >> pshift) == prefix))
                    b = (key >> shift) & (nb - 1);
                if (__any_sync(0xffffffffu, b != 0xFFFFFFFFu)) {
                    const uint32_t grp = __match_any_sync(0xffffffffu, b);  // warp-aggregated
                    if (b != 0xFFFFFFFFu && (__ffs(grp) - 1) == (tid & 31))
                        atomicAdd(&hist[b], (uint32_t)__popc(grp));
                }
            }
            cluster.sync();
            uint32_t mc = 0;
            if (tid < per) {
                const int b = rank * per + tid;
                for (int r = 0; r < CL; ++r) mc += cluster.map_shared_rank(hist, r)[b];
                m_cnt[tid] = mc;
            }
            const uint32_t rc = block_sum<uint32_t, BS>(mc);
            if (tid == 0) range_cnt = rc;
            cluster.sync();
            if (tid == 0) {  // descending over ranks: higher ranks hold higher buckets
                uint32_t above = 0;
                int rstar = -1;
                for (int r = CL - 1; r >= 0; --r) {
                    const uint32_t cr = *cluster.map_shared_rank(&range_cnt, r);
                    if (above < need && need <= above + cr) {
                        rstar = r;
                        break;
                    }
                    above += cr;
                }
                s_rstar = rstar;
                s_above_r = above;
            }
            __syncthreads();
            if (rank == s_rstar) {
                const int bi = per - 1 - tid;
                const uint32_t c0 = (tid < per) ? m_cnt[bi] : 0;
                uint32_t ctot;
                const uint32_t above = block_excl_scan<uint32_t, BS>(c0, &ctot) + s_above_r;
                if (tid < per && above < need && need <= above + c0) {
                    for (int r = 0; r < CL; ++r) {
                        *cluster.map_shared_rank(&res_bucket, r) = (uint32_t)(rank * per + bi);
                        *cluster.map_shared_rank(&res_above, r) = above;
                    }
                }
            }
            cluster.sync();
            prefix = (prefix << bits) | res_bucket;
            need -= res_above;
            cluster.sync();
        }
    }
    const uint32_t vstar = prefix;
    const bool has_thr = n_free > 0;
    const int take_eq = has_thr ? (int)need : 0;
    int fg = 0, eq = 0;
    for (int i = tid; i < n_loc; i += BS) {
        const uint32_t key = keys[i];
        if (key == kForcedKey || (has_thr && key > vstar)) ++fg;
        else if (has_thr && key == vstar) ++eq;
    }
    fg = block_sum<int, BS>(fg);
    eq = block_sum<int, BS>(eq);
    if (tid == 0) {
        slice_fg = fg;
        slice_eq = eq;
    }
    cluster.sync();
    int base_pos = 0, base_eq = 0;
    for (int r = 0; r < rank; ++r) {
        const int fr = *cluster.map_shared_rank(&slice_fg, r);
        const int er = *cluster.map_shared_rank(&slice_eq, r);
        base_pos += fr + max(0, min(er, take_eq - base_eq));
        base_eq += er;
    }
    cluster.sync();  // remote reads done before any CTA may exit
    // ---- ordered compaction: warp ballots + one block scan per 8-item chunk ----
    int32_t* idx_h = idx + (size_t)h * L;
    int32_t* inv_h = inv ? inv + (size_t)h * L : nullptr;
    constexpr int IPT = 8;
    for (int c0 = 0; c0 < n_loc; c0 += BS * IPT) {
        uint32_t kbits = 0, ebits = 0;
        int neq = 0;
#pragma unroll
        for (int u = 0; u < IPT; ++u) {
            const int i = c0 + tid * IPT + u;
            if (i < n_loc) {
                const uint32_t key = keys[i];
                if (key == kForcedKey || (has_thr && key > vstar)) kbits |= 1u << u;
                else if (has_thr && key == vstar) {
                    ebits |= 1u << u;
                    ++neq;
                }
            }
        }
        int eq_total;
        int running_eq = block_excl_scan<int, BS>(neq, &eq_total) + base_eq;
#pragma unroll
        for (int u = 0; u < IPT; ++u)
            if ((ebits >> u & 1u) && running_eq++ < take_eq) kbits |= 1u << u;
        int keep_total;
        int pos = block_excl_scan<int, BS>(__popc(kbits), &keep_total) + base_pos;
#pragma unroll
        for (int u = 0; u < IPT; ++u) {
            const int i = c0 + tid * IPT + u;
            if (i >= n_loc) break;
            const int t = t_begin + i;
            if (kbits >> u & 1u) {
                idx_h[pos] = t;
                if (inv_h) inv_h[t] = pos;
                ++pos;
            } else if (inv_h) {
                inv_h[t] = -1;
            }
        }
        base_pos += keep_total;
        base_eq += eq_total;
    }
}

}  // namespace

static void launch_budget_kernel(const float* v, int L, double tau, int min_keep, int32_t* k_keep,
                                 int32_t* status, int mode, float* sl_out, int exact_total,
                                 cudaStream_t st) {
    const int slice = (L + CL - 1) / CL;
    if (slice <= kSliceMax) {
        ensure_smem_attr(reinterpret_cast<const void*>(budget_kernel<true>),
                         kSliceMax * 4 + 4 * 2048 * 4);
        const int smem = (slice + 3) / 4 * 4 * 4 + 4 * 2048 * 4;  // slice + mass limbs
        budget_kernel<true><<<CL, BB, smem, st>>>(v, L, tau, min_keep, k_keep, status, mode,
                                                  sl_out, exact_total);
    } else {
        budget_kernel<false><<<CL, BB, 0, st>>>(v, L, tau, min_keep, k_keep, status, mode, sl_out,
                                                exact_total);
    }
}

int launch_write_int(int32_t* dst, int32_t value, cudaStream_t st) {
    write_int_kernel<<<1, 1, 0, st>>>(dst, value);
    TSA_LAUNCH_CHECK("write_int");
    return 0;
}

int launch_budget(const tsa_desc& d, const float* s, int32_t* k_keep, float* headsum,
                  int32_t* status, int min_keep, cudaStream_t st) {
    const int L = d.seq_len;
    headsum_kernel<<<(L + 255) / 256, 256, 0, st>>>(s, headsum, d.n_heads, L);
    TSA_LAUNCH_CHECK("headsum");
    launch_budget_kernel(headsum, L, d.tau, min_keep, k_keep, status, BUDGET_FROM_HEADSUM, nullptr,
                         scoring_mode(d) == TSA_SCORING_REFERENCE ? 1 : 0, st);
    TSA_LAUNCH_CHECK("budget");
    return 0;
}

int launch_aggregate(const tsa_desc& d, const float* s, float* sl, float* headsum,
                     int32_t* status, cudaStream_t st) {
    const int L = d.seq_len;
    headsum_kernel<<<(L + 255) / 256, 256, 0, st>>>(s, headsum, d.n_heads, L);
    TSA_LAUNCH_CHECK("headsum");
    launch_budget_kernel(headsum, L, 0.0, 1, nullptr, status, AGGREGATE_ONLY, sl,
                         scoring_mode(d) == TSA_SCORING_REFERENCE ? 1 : 0, st);
    TSA_LAUNCH_CHECK("aggregate");
    return 0;
}

int launch_coverage_from_sl(const tsa_desc& d, const float* sl, int32_t* k_keep, int32_t* status,
                            int min_keep, cudaStream_t st) {
    launch_budget_kernel(sl, d.seq_len, d.tau, min_keep, k_keep, status, BUDGET_FROM_SL, nullptr, 1,
                         st);
    TSA_LAUNCH_CHECK("coverage_budget");
    return 0;
}

int launch_select(const tsa_desc& d, const float* s, const int32_t* k_keep, const int32_t* forced,
                  int32_t n_forced, int32_t forced_begin, int32_t* idx, int32_t* inv,
                  cudaStream_t st) {
    const int nh = d.head_end - d.head_begin;
    const int slice = (d.seq_len + CL - 1) / CL;
    if (slice <= kSliceMax) {
        const int smem = slice * 4;
        ensure_smem_attr(reinterpret_cast<const void*>(select_smem_kernel), kSliceMax * 4);
        select_smem_kernel<<<dim3(CL, nh), BS, smem, st>>>(s, d.seq_len, k_keep, forced, n_forced,
                                                           forced_begin, d.head_begin, idx, inv);
    } else {
        select_kernel<<<dim3(CL, nh), BT, 0, st>>>(s, d.seq_len, k_keep, forced, n_forced,
                                                   forced_begin, d.head_begin, idx, inv);
    }
    TSA_LAUNCH_CHECK("select");
    return 0;
}

}  // namespace tsa
