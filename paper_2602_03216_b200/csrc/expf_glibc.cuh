// expf as the reference's std::exp(float) computes it, bit for bit.
//
// The reference's masked softmax (tensor_ops.cpp:59-65) calls std::exp on a
// float, i.e. glibc's expf.  glibc >= 2.27 implements it in double precision
// (sysdeps/ieee754/flt-32/e_expf.c): x*N/ln2 = k + r, 2^(k/N) from a 32-entry
// table, a cubic in r, one rounding to float at the end -- so a GPU port of
// the same double arithmetic reproduces it exactly.  The table and
// coefficients below are glibc's __exp2f_data (N = 32); the contraction
// pattern (r = fma(InvLn2N, x, -kd), fused polynomial) is the x86-64 FMA
// variant the reference binary dispatches to.  Checked against the host libm
// on every float in [-104, -0] (1,120,927,745 inputs, 0 mismatches:
// tools/probes/expf_glibc_exhaustive.c, profiles/r2/expf_glibc_exhaustive.log)
// and on the GPU against the oracle's libm (tests/test_gpu_exact.py).
//
// Domain: the softmax argument x - max <= 0.  Below log(2^-150) glibc returns
// +0 (its underflow branch); NaN / +inf inputs never reach this function.
#pragma once

#include <cstdint>

namespace tsa_dev {

__device__ __constant__ const uint64_t kExp2fTab[32] = {
    0x3ff0000000000000ull, 0x3fefd9b0d3158574ull, 0x3fefb5586cf9890full, 0x3fef9301d0125b51ull,
    0x3fef72b83c7d517bull, 0x3fef54873168b9aaull, 0x3fef387a6e756238ull, 0x3fef1e9df51fdee1ull,
    0x3fef06fe0a31b715ull, 0x3feef1a7373aa9cbull, 0x3feedea64c123422ull, 0x3feece086061892dull,
    0x3feebfdad5362a27ull, 0x3feeb42b569d4f82ull, 0x3feeab07dd485429ull, 0x3feea47eb03a5585ull,
    0x3feea09e667f3bcdull, 0x3fee9f75e8ec5f74ull, 0x3feea11473eb0187ull, 0x3feea589994cce13ull,
    0x3feeace5422aa0dbull, 0x3feeb737b0cdc5e5ull, 0x3feec49182a3f090ull, 0x3feed503b23e255dull,
    0x3feee89f995ad3adull, 0x3feeff76f2fb5e47ull, 0x3fef199bdd85529cull, 0x3fef3720dcef9069ull,
    0x3fef5818dcfba487ull, 0x3fef7c97337b9b5full, 0x3fefa4afa2a490daull, 0x3fefd0765b6e4540ull,
};

// InvLn2N, C0, C1, C2 from constant memory: DFMA reads them as c[][]
// operands (as immediates they would be rebuilt with MOV pairs per call).
__device__ __constant__ double kExpfC[4] = {  // not const: no folding into immediates
    0x1.71547652b82fep+0 * 32, 0x1.c6af84b912394p-5 / 32 / 32 / 32, 0x1.ebfce50fac4f3p-3 / 32 / 32,
    0x1.62e42ff0c52d6p-1 / 32};

// Call sites keep the table in shared memory (exp2f_table_to_smem): indexed
// per thread, a __constant__ table would serialise a warp's distinct lookups.
__device__ __forceinline__ void exp2f_table_to_smem(uint64_t* tab) {
    for (int i = threadIdx.x; i < 32; i += blockDim.x) tab[i] = kExp2fTab[i];
}

// Branch-free (the underflow case is a select at the end), so a thread's
// independent exponentials interleave.
__device__ __forceinline__ float expf_glibc(float x, const uint64_t* __restrict__ tab) {
    const double kInvLn2N = kExpfC[0], kC0 = kExpfC[1], kC1 = kExpfC[2], kC2 = kExpfC[3];
    constexpr double kShift = 0x1.8p+52;
    const double xd = (double)fmaxf(x, -104.0f);  // keeps the table index in range
    double kd = __fma_rn(kInvLn2N, xd, kShift);  // round(x N / ln2) in the low mantissa bits
    const uint64_t ki = (uint64_t)__double_as_longlong(kd);
    kd = __dsub_rn(kd, kShift);
    const double r = __fma_rn(kInvLn2N, xd, -kd);
    const uint64_t t = tab[ki & 31] + (ki << 47);
    const double s = __longlong_as_double((long long)t);
    const double z = __fma_rn(kC0, r, kC1);
    const double r2 = __dmul_rn(r, r);
    double y = __fma_rn(kC2, r, 1.0);
    y = __fma_rn(z, r2, y);
    y = __dmul_rn(y, s);
    // x < log(2^-150): glibc's __math_uflowf -> +0
    return x < -0x1.9fe368p6f ? 0.0f : __double2float_rn(y);
}

}  // namespace tsa_dev
