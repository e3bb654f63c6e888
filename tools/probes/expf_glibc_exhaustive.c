/* Exhaustive check of the double-precision expf port used by the GPU
 * scorer (paper_2602_03216_b200/csrc/expf_glibc.cuh) against the host libm's
 * expf -- the function the reference's softmax calls (tensor_ops.cpp:62).
 * Every float in [-104, -0] (the softmax argument x - max <= 0).
 *   gcc -O2 -ffp-contract=off expf_glibc_exhaustive.c -lm && ./a.out          */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

static uint64_t T[32];

static float port(float x) {
    if (x < -0x1.9fe368p6f) return 0.0f;
    const double kInvLn2N = 0x1.71547652b82fep+0 * 32, kShift = 0x1.8p+52;
    const double C0 = 0x1.c6af84b912394p-5 / 32 / 32 / 32, C1 = 0x1.ebfce50fac4f3p-3 / 32 / 32,
                 C2 = 0x1.62e42ff0c52d6p-1 / 32;
    double xd = x, kd = fma(kInvLn2N, xd, kShift), s, r, z, r2, y;
    uint64_t ki, t;
    memcpy(&ki, &kd, 8);
    kd -= kShift;
    r = fma(kInvLn2N, xd, -kd);
    t = T[ki & 31] + (ki << 47);
    memcpy(&s, &t, 8);
    z = fma(C0, r, C1);
    r2 = r * r;
    y = fma(C2, r, 1.0);
    y = fma(z, r2, y);
    return (float)(y * s);
}

int main(void) {
    for (int i = 0; i < 32; i++) {
        double v = exp2((double)i / 32);
        uint64_t u;
        memcpy(&u, &v, 8);
        T[i] = u - ((uint64_t)i << 47);
    }
    long bad = 0, n = 0;
    for (uint32_t u = 0x80000000u;; ++u) {  /* -0 .. -104 */
        float x, a, b;
        uint32_t ua, ub;
        memcpy(&x, &u, 4);
        a = expf(x);
        b = port(x);
        memcpy(&ua, &a, 4);
        memcpy(&ub, &b, 4);
        ++n;
        if (ua != ub && bad++ < 10) printf("mismatch x=%a libm=%a port=%a\n", x, a, b);
        if (u == 0xC2D00000u) break;
    }
    printf("inputs %ld mismatches %ld\n", n, bad);
    return bad != 0;
}
