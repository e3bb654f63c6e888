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
// K3 (select_tokens, token_coverage.cpp:111-152), one CTA per head:
//   radix select of the (k - |F|)-th largest non-forced score, then one
//   ordered compaction pass: keep t if forced, if s > v*, or if s == v* and t
//   is among the lowest-index (k - |F| - count(> v*)) ties.  Output is
//   ascending by construction; the inverse map is written in the same pass.
#include "common.cuh"

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
template <typename U>
__device__ U block_excl_scan(U v, U* total) {
    __shared__ U warp_sums[BT / 32];
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
        U w = warp_sums[lane];
        U wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const U n = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += n;
        }
        warp_sums[lane] = wi - w;  // exclusive prefix of warp totals
    }
    __syncthreads();
    const U excl = warp_sums[warp] + incl - v;
    // total = exclusive prefix of the last warp + its inclusive sum
    __shared__ U s_total;
    if (threadIdx.x == BT - 1) s_total = excl + v;
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

__global__ void __launch_bounds__(BT) budget_kernel(const float* __restrict__ headsum, int L,
                                                    double tau, int min_keep,
                                                    int32_t* __restrict__ k_keep,
                                                    int32_t* __restrict__ status, int mode,
                                                    float* __restrict__ sl_out, int exact_total) {
    __shared__ float stage[2][2048];
    __shared__ float s_total;
    __shared__ uint32_t hist_cnt[2048];
    __shared__ unsigned long long hist_mass[2048];
    __shared__ uint32_t s_prefix;
    __shared__ unsigned long long s_mass_below;
    __shared__ uint32_t s_cnt_below;
    __shared__ int s_done;

    const int tid = threadIdx.x;
    float total = 1.0f;
    if (mode != BUDGET_FROM_SL) {
    if (exact_total) {
    // ---- total: sequential f32 chain (token_coverage.cpp:58-61) ----
    // Warps stage 2048-float chunks into a double buffer; thread 0 consumes
    // them with 16-B shared loads kept ahead of the dependent FADD chain.
    constexpr int CH = 2048;
    const int nchunk = (L + CH - 1) / CH;
    for (int i = tid; i < CH; i += BT) stage[0][i] = i < L ? headsum[i] : 0.0f;
    __syncthreads();
    total = 0.0f;
    for (int c = 0; c < nchunk; ++c) {
        if (c + 1 < nchunk) {
            const int base = (c + 1) * CH;
            for (int i = tid; i < CH; i += BT)
                stage[(c + 1) & 1][i] = base + i < L ? headsum[base + i] : 0.0f;
        }
        if (tid == 0) {
            const float* buf = stage[c & 1];
            const int n = min(CH, L - c * CH);
            const float4* b4 = reinterpret_cast<const float4*>(buf);
            const int n4 = n / 4;
#pragma unroll 8
            for (int i = 0; i < n4; ++i) {
                const float4 v = b4[i];
                total = __fadd_rn(total, v.x);
                total = __fadd_rn(total, v.y);
                total = __fadd_rn(total, v.z);
                total = __fadd_rn(total, v.w);
            }
            for (int i = n4 * 4; i < n; ++i) total = __fadd_rn(total, buf[i]);
        }
        __syncthreads();
    }
    } else {
    // ---- total: deterministic parallel reduction in f64 (FAST scoring mode) ----
    // Fixed thread->element assignment and a fixed reduction tree, so the
    // result is reproducible; it differs from the sequential f32 chain by far
    // less than the FAST scores differ from reference-order scores.
    __shared__ double red[BT / 32];
    double acc = 0.0;
    for (int t = tid; t < L; t += BT) acc += (double)headsum[t];
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((tid & 31) == 0) red[tid >> 5] = acc;
    __syncthreads();
    if (tid < 32) {
        double w = red[tid];
#pragma unroll
        for (int o = 16; o; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
        if (tid == 0) total = (float)w;
    }
    }
    if (tid == 0) s_total = total;
    __syncthreads();
    total = s_total;
    if (!(total > 0.0f)) {  // aggregate_scores throws (:62-64)
        if (tid == 0) {
            *status = 1;
            if (k_keep) *k_keep = min_keep;
        }
        return;
    }
    if (mode == AGGREGATE_ONLY) {
        for (int t = tid; t < L; t += BT) sl_out[t] = __fdiv_rn(headsum[t], total);
        return;
    }
    }  // mode != BUDGET_FROM_SL
    // ---- coverage crossing ----
    // T = ceil(tau * 2^62); tau = 0 -> k_sparse = 0 (prefix 0 >= 0, :82).
    const double tscaled = ldexp(tau, 62);
    unsigned long long T = (unsigned long long)tscaled;
    if ((double)T < tscaled) ++T;
    if (T == 0ull) {
        if (tid == 0) *k_keep = max(L, min_keep);
        return;
    }
    if (tid == 0) {
        s_prefix = 0;
        s_mass_below = 0;
        s_cnt_below = 0;
        s_done = 0;
    }
    for (int lvl = 0; lvl < 3; ++lvl) {
        const int shift = kShift[lvl], nb = 1 << kBits[lvl];
        for (int b = tid; b < nb; b += BT) {
            hist_cnt[b] = 0;
            hist_mass[b] = 0;
        }
        __syncthreads();
        const uint32_t prefix = s_prefix;
        const int pshift = shift + kBits[lvl];
        // warp-aggregated: lanes hitting the same bucket combine their count and
        // mass (three 21-bit limbs so the 32-lane sums cannot overflow) before
        // one shared atomic per distinct bucket
        for (int base = 0; base < L; base += BT) {
            const int t = base + tid;
            uint32_t b = 0xFFFFFFFFu;
            unsigned long long m = 0;
            if (t < L) {
                const float sl = __fdiv_rn(headsum[t], total);
                const uint32_t key = score_key(sl);
                if (pshift >= 32 || (key >> pshift) == prefix) {
                    b = (key >> shift) & (nb - 1);
                    m = (unsigned long long)ldexp((double)sl, 62);
                }
            }
            const uint32_t grp = __match_any_sync(0xffffffffu, b);
            const uint32_t l0 = __reduce_add_sync(grp, (uint32_t)(m & 0x1FFFFFu));
            const uint32_t l1 = __reduce_add_sync(grp, (uint32_t)((m >> 21) & 0x1FFFFFu));
            const uint32_t l2 = __reduce_add_sync(grp, (uint32_t)(m >> 42));
            if (b != 0xFFFFFFFFu && (__ffs(grp) - 1) == (int)(tid & 31)) {
                const unsigned long long sum = (unsigned long long)l0 +
                                               ((unsigned long long)l1 << 21) +
                                               ((unsigned long long)l2 << 42);
                atomicAdd(&hist_cnt[b], (uint32_t)__popc(grp));
                atomicAdd(&hist_mass[b], sum);
            }
        }
        __syncthreads();
        // exclusive scan over buckets (2 buckets per thread, ascending)
        const int b0 = 2 * tid, b1 = 2 * tid + 1;
        unsigned long long m0 = b0 < nb ? hist_mass[b0] : 0, m1 = b1 < nb ? hist_mass[b1] : 0;
        uint32_t c0 = b0 < nb ? hist_cnt[b0] : 0, c1 = b1 < nb ? hist_cnt[b1] : 0;
        unsigned long long mtot;
        uint32_t ctot;
        const unsigned long long mex = block_excl_scan<unsigned long long>(m0 + m1, &mtot);
        const uint32_t cex = block_excl_scan<uint32_t>(c0 + c1, &ctot);
        const unsigned long long need = T - s_mass_below;  // > 0
        __syncthreads();
        if (lvl == 0 && mtot < need) {
            // total mass never reaches tau: k_sparse = L
            if (tid == 0) s_done = 1;
        } else {
            // bucket b with excl[b] < need <= excl[b] + mass[b]
            if (b0 < nb && mex < need && need <= mex + m0) {
                s_prefix = (prefix << kBits[lvl]) | (uint32_t)b0;
                s_mass_below += mex;
                s_cnt_below += cex;
            }
            if (b1 < nb && mex + m0 < need && need <= mex + m0 + m1) {
                s_prefix = (prefix << kBits[lvl]) | (uint32_t)b1;
                s_mass_below += mex + m0;
                s_cnt_below += cex + c0;
            }
        }
        __syncthreads();
        if (s_done) break;
    }
    if (tid == 0) {
        int k_sparse = L;
        if (!s_done) {
            const float v = __uint_as_float(s_prefix);
            const unsigned long long m = (unsigned long long)ldexp((double)v, 62);
            const unsigned long long need = T - s_mass_below;
            const unsigned long long c = (need + m - 1) / m;  // m > 0: bucket mass crossed
            k_sparse = (int)(s_cnt_below + c);
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

__global__ void __launch_bounds__(BT) select_kernel(const float* __restrict__ s, int L,
                                                    const int32_t* __restrict__ k_keep_p,
                                                    const int32_t* __restrict__ forced, int nf,
                                                    int fbegin, int head_begin,
                                                    int32_t* __restrict__ idx,
                                                    int32_t* __restrict__ inv) {
    __shared__ uint32_t hist[2048];
    __shared__ uint32_t s_prefix, s_cnt_gt, s_need;
    const int h = head_begin + blockIdx.x;
    const int tid = threadIdx.x;
    const float* sh = s + (size_t)h * L;
    const int k_keep = *k_keep_p;
    const int n_free = k_keep - nf;
    if (tid == 0) {
        s_prefix = 0;
        s_cnt_gt = 0;
        s_need = (uint32_t)max(n_free, 0);
    }
    __syncthreads();
    // ---- radix select of the n_free-th largest non-forced key ----
    if (n_free > 0) {
        for (int lvl = 0; lvl < 3; ++lvl) {
            const int shift = kShift[lvl], nb = 1 << kBits[lvl];
            const int pshift = shift + kBits[lvl];
            for (int b = tid; b < nb; b += BT) hist[b] = 0;
            __syncthreads();
            const uint32_t prefix = s_prefix;
            for (int base = 0; base < L; base += BT) {
                const int t = base + tid;
                uint32_t b = 0xFFFFFFFFu;
                if (t < L && !is_forced(t, forced, nf, fbegin)) {
                    const uint32_t key = score_key(sh[t]);
                    if (pshift >= 32 || (key >> pshift) == prefix) b = (key >> shift) & (nb - 1);
                }
                const uint32_t grp = __match_any_sync(0xffffffffu, b);  // warp-aggregated
                if (b != 0xFFFFFFFFu && (__ffs(grp) - 1) == (tid & 31))
                    atomicAdd(&hist[b], (uint32_t)__popc(grp));
            }
            __syncthreads();
            // descending: count of keys in buckets above b = exclusive scan from the top
            const int b0 = nb - 1 - 2 * tid, b1 = nb - 2 - 2 * tid;  // thread handles 2, top-down
            const uint32_t c0 = b0 >= 0 ? hist[b0] : 0, c1 = b1 >= 0 ? hist[b1] : 0;
            uint32_t ctot;
            const uint32_t above = block_excl_scan<uint32_t>(c0 + c1, &ctot);
            const uint32_t need = s_need;
            __syncthreads();
            if (b0 >= 0 && above < need && need <= above + c0) {
                s_prefix = (prefix << kBits[lvl]) | (uint32_t)b0;
                s_cnt_gt += above;
                s_need = need - above;
            }
            if (b1 >= 0 && above + c0 < need && need <= above + c0 + c1) {
                s_prefix = (prefix << kBits[lvl]) | (uint32_t)b1;
                s_cnt_gt += above + c0;
                s_need = need - above - c0;
            }
            __syncthreads();
        }
    }
    const uint32_t vstar = s_prefix;
    // ties to take at v* (lowest index first); with n_free == 0 none
    const int take_eq = n_free > 0 ? (int)s_need : 0;
    const bool has_thr = n_free > 0;
    // ---- ordered compaction ----
    int32_t* idx_h = idx + (size_t)h * L;
    int32_t* inv_h = inv ? inv + (size_t)h * L : nullptr;
    int base_pos = 0, base_eq = 0;
    constexpr int IPT = 4;
    for (int t0 = 0; t0 < L; t0 += BT * IPT) {
        int keep_flags = 0, eq_flags = 0, nkeep = 0, neq = 0;
        uint32_t keys[IPT];
        bool forced_f[IPT];
#pragma unroll
        for (int i = 0; i < IPT; ++i) {
            const int t = t0 + tid * IPT + i;
            forced_f[i] = false;
            keys[i] = 0;
            if (t < L) {
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
            if (t >= L) continue;
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
            if (t >= L) continue;
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

}  // namespace

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
    budget_kernel<<<1, BT, 0, st>>>(headsum, L, d.tau, min_keep, k_keep, status,
                                    BUDGET_FROM_HEADSUM, nullptr,
                                    scoring_mode(d) == TSA_SCORING_REFERENCE ? 1 : 0);
    TSA_LAUNCH_CHECK("budget");
    return 0;
}

int launch_aggregate(const tsa_desc& d, const float* s, float* sl, float* headsum,
                     int32_t* status, cudaStream_t st) {
    const int L = d.seq_len;
    headsum_kernel<<<(L + 255) / 256, 256, 0, st>>>(s, headsum, d.n_heads, L);
    TSA_LAUNCH_CHECK("headsum");
    budget_kernel<<<1, BT, 0, st>>>(headsum, L, 0.0, 1, nullptr, status, AGGREGATE_ONLY, sl,
                                    scoring_mode(d) == TSA_SCORING_REFERENCE ? 1 : 0);
    TSA_LAUNCH_CHECK("aggregate");
    return 0;
}

int launch_coverage_from_sl(const tsa_desc& d, const float* sl, int32_t* k_keep, int32_t* status,
                            int min_keep, cudaStream_t st) {
    budget_kernel<<<1, BT, 0, st>>>(sl, d.seq_len, d.tau, min_keep, k_keep, status, BUDGET_FROM_SL,
                                    nullptr, 1);
    TSA_LAUNCH_CHECK("coverage_budget");
    return 0;
}

int launch_select(const tsa_desc& d, const float* s, const int32_t* k_keep, const int32_t* forced,
                  int32_t n_forced, int32_t forced_begin, int32_t* idx, int32_t* inv,
                  cudaStream_t st) {
    const int nh = d.head_end - d.head_begin;
    select_kernel<<<nh, BT, 0, st>>>(s, d.seq_len, k_keep, forced, n_forced, forced_begin,
                                     d.head_begin, idx, inv);
    TSA_LAUNCH_CHECK("select");
    return 0;
}

}  // namespace tsa
