// FFMA2 issue rate of the exact scorer's inner-product pattern (q scalar
// broadcast into both halves, key pair, 64-bit accumulator) at 1..4 warps per
// scheduler, with and without bf16->f32 PRMT conversions in the stream.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 ffma2_probe.cu -o ffma2_probe
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t f2(float a, float b) {
    uint64_t r;
    asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t d;
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}

template <bool CONV, int ORDER>
__global__ void k(float* out, int iters, const uint32_t* kin) {
    uint64_t acc[8][4];
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0;
    float q[8];
    uint32_t w[8];
#pragma unroll
    for (int a = 0; a < 8; ++a) {
        q[a] = 1.0f + threadIdx.x * 1e-3f + a;
        w[a] = kin[(threadIdx.x + a) & 63];
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int pp = 0; pp < 4; ++pp) {
            uint64_t kp[4];
#pragma unroll
            for (int i2 = 0; i2 < 4; ++i2) {
                if (CONV)
                    kp[i2] = (pp & 1) ? f2(__uint_as_float(__byte_perm(w[2 * i2], 0, 0x3244)),
                                           __uint_as_float(__byte_perm(w[2 * i2 + 1], 0, 0x3244)))
                                      : f2(__uint_as_float(__byte_perm(w[2 * i2], 0, 0x1044)),
                                           __uint_as_float(__byte_perm(w[2 * i2 + 1], 0, 0x1044)));
                else
                    kp[i2] = f2(__uint_as_float(w[2 * i2]), __uint_as_float(w[2 * i2 + 1]));
            }
            if (ORDER == 0) {
#pragma unroll
                for (int a = 0; a < 8; ++a)
#pragma unroll
                    for (int i2 = 0; i2 < 4; ++i2) acc[a][i2] = fma2(f2(q[a], q[a]), kp[i2], acc[a][i2]);
            } else if (ORDER == 1) {
#pragma unroll
                for (int i2 = 0; i2 < 4; ++i2)
#pragma unroll
                    for (int a = 0; a < 8; ++a) acc[a][i2] = fma2(f2(q[a], q[a]), kp[i2], acc[a][i2]);
            } else {  // scalar FFMA, same work
#pragma unroll
                for (int a = 0; a < 8; ++a)
#pragma unroll
                    for (int i2 = 0; i2 < 4; ++i2) {
                        float lo, hi, k0, k1;
                        asm("mov.b64 {%0,%1}, %2;" : "=f"(lo), "=f"(hi) : "l"(acc[a][i2]));
                        asm("mov.b64 {%0,%1}, %2;" : "=f"(k0), "=f"(k1) : "l"(kp[i2]));
                        asm volatile("fma.rn.f32 %0, %1, %2, %0;" : "+f"(lo) : "f"(q[a]), "f"(k0));
                        asm volatile("fma.rn.f32 %0, %1, %2, %0;" : "+f"(hi) : "f"(q[a]), "f"(k1));
                        acc[a][i2] = f2(lo, hi);
                    }
            }
#pragma unroll
            for (int a = 0; a < 8; ++a) w[a] = w[a] * 1664525u + 1013904223u;
        }
    }
    float s = 0;
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) s += __uint_as_float((uint32_t)acc[a][b]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    float* out;
    uint32_t* kin;
    cudaMalloc(&out, 148 * 1024 * 4);
    cudaMalloc(&kin, 64 * 4);
    cudaMemset(kin, 0x3f, 256);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 20000;
    for (int order = 0; order < 3; ++order)
        for (int warps = 8; warps <= 16; warps += 8) {
            auto fn = order == 0 ? k<true, 0> : order == 1 ? k<true, 1> : k<true, 2>;
            fn<<<148, warps * 32>>>(out, 10, kin);
            cudaEventRecord(a);
            fn<<<148, warps * 32>>>(out, iters, kin);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            const double fma = 148.0 * warps * 32 * iters * 4 * 32 * 2;
            printf("order %d warps/SM %2d: %.3f ms  %.1f FMA/clk/SM at 1.965 GHz\n", order, warps, ms,
                   fma / (ms * 1e-3) / 148 / 1.965e9);
        }
    return 0;
}
