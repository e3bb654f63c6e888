// Throughput probe of single-CTA tcgen05.mma (kind::f16, bf16 -> f32) shapes
// used by the attention kernel: cycles per instruction (K = 16) when one
// thread issues a long back-to-back stream, on every SM at once.
//   mode 0: SS, A and B K-major SW128, M=128, N=n      (S = Q K^T)
//   mode 1: TS, A in TMEM, B MN-major SW128, M=128, N=n (O = P V)
// usage: umma_rate   (prints cycles/UMMA per mode and N)
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "../../paper_2602_03216_b200/csrc/sm100.cuh"

using namespace tsa_dev;

struct __align__(1024) Smem {
    uint8_t a[2 * 16384];
    uint8_t b[2 * 32768];
    uint64_t bar;
    uint32_t tmem;
};

__device__ volatile int g_stop;
__device__ int g_rand;
// interference: 0 none, 1 warps 1..3 stream tcgen05.ld of TMEM columns [384, 512),
// 2 warps 1..3 stream tcgen05.st there, 3 warps 1..3 stream shared-memory stores
__global__ void __launch_bounds__(384, 1) rate_kernel(int mode, int n, int reps, long long* out,
                                                      int interf) {
    extern __shared__ uint8_t raw[];
    Smem& s = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    const uint32_t warp = warp_id_uniform();
    // random bf16 pairs in [-1, 1) (data-dependent power / throughput)
    auto rnd = [](uint32_t i) {
        uint32_t h = i * 2654435761u ^ 0x9E3779B9u;
        h ^= h >> 15; h *= 0x85EBCA6Bu; h ^= h >> 13;
        const float f0 = ((h & 0xFFFF) / 32768.0f) - 1.0f, f1 = ((h >> 16) / 32768.0f) - 1.0f;
        return pack_bf16x2(f0, f1);
    };
    for (int i = threadIdx.x; i < (int)sizeof(s.a) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(s.a)[i] = g_rand ? rnd(i) : 0;
    for (int i = threadIdx.x; i < (int)sizeof(s.b) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(s.b)[i] = g_rand ? rnd(i + 77777) : 0;
    if (threadIdx.x == 0) {
        mbar_init(&s.bar, 1);
        fence_barrier_init();
    }
    fence_proxy_async_smem();
    if (warp == 0) tmem_alloc(&s.tmem, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (interf >= 4 && warp > 0 && (warp & 3) == 0) {
        // same sub-partition as the issuing warp 0: a MUFU- (4) or FMA-heavy (5) stream
        float x0 = threadIdx.x * 1e-3f, x1 = x0 + 1.0f, x2 = x0 + 2.0f, x3 = x0 + 3.0f;
        for (int it = 0; it < reps * 64 && !g_stop; ++it) {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                if (interf == 4) {
                    x0 = ex2_approx(x0 * -0.5f); x1 = ex2_approx(x1 * -0.5f);
                    x2 = ex2_approx(x2 * -0.5f); x3 = ex2_approx(x3 * -0.5f);
                } else {
                    x0 = fmaf(x0, 0.999f, 0.001f); x1 = fmaf(x1, 0.999f, 0.001f);
                    x2 = fmaf(x2, 0.999f, 0.001f); x3 = fmaf(x3, 0.999f, 0.001f);
                }
            }
        }
        if (x0 + x1 + x2 + x3 == 12345.f) out[0] = 0;
    }
    if (interf > 0 && interf < 4 && warp > 0 && warp < 4) {
        const uint32_t lane_off = ((warp & 3) * 32) << 16;
        uint32_t r[32];
        for (int i = 0; i < 32; ++i) r[i] = i;
        uint32_t acc = 0;
        for (int it = 0; it < reps * 4; ++it) {
            if (interf == 1) {
                tmem_ld32(s.tmem + 384 + (it & 3) * 32 + lane_off, r);
                tmem_wait_ld();
                acc += r[it & 31];
            } else if (interf == 2) {
                tmem_st32(s.tmem + 384 + (it & 3) * 32 + lane_off, r);
                tmem_wait_st();
            } else {
                reinterpret_cast<volatile uint32_t*>(s.a)[(threadIdx.x + it * 128) & 4095] = it;
            }
            if (g_stop) break;
        }
        if (acc == 12345) out[0] = 0;
    }
    if (threadIdx.x == 0) {
        const uint32_t idesc = idesc_bf16_f32(128, n, 0, mode == 1 ? 1 : 0);
        const uint32_t a = smem_u32(s.a), b = smem_u32(s.b);
        const uint32_t d = s.tmem;          // columns [0, n)
        const uint32_t pa = s.tmem + 256;   // A operand in TMEM for mode 1
        const uint64_t da = sdesc_kmajor_sw128(a), db = sdesc_kmajor_sw128(b),
                       dv = sdesc_mnmajor_sw128(b, 16384);
        long long t0 = clock64();
        if (mode == 0) {
            for (int r = 0; r < reps; ++r) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    mma_bf16_ss(d, da + (((kk >> 2) * 16384 + (kk & 3) * 32) >> 4),
                                db + (((kk >> 2) * 32768 + (kk & 3) * 32) >> 4), idesc, 1u);
            }
        } else {
            for (int r = 0; r < reps; ++r) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    mma_bf16_ts(d, pa + kk * 8, dv + ((kk * 2048) >> 4), idesc, 1u);
            }
        }
        mma_commit(&s.bar);
        mbar_wait(&s.bar, 0);
        long long t1 = clock64();
        out[blockIdx.x] = t1 - t0;
        g_stop = 1;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(s.tmem, 512);
}

int main() {
    long long* d_out;
    cudaMalloc(&d_out, 148 * sizeof(long long));
    const int smem = sizeof(Smem) + 1024;
    cudaFuncSetAttribute(rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int reps = 4000;
    for (int rnd : {1}) for (int interf : {0})
    for (int mode = 0; mode < 2; ++mode) {
        for (int n : {64, 128}) {
            int zero = 0;
            cudaMemcpyToSymbol(g_rand, &rnd, 4);
            cudaMemcpyToSymbol(g_stop, &zero, 4);
            rate_kernel<<<148, 384, smem>>>(mode, n, reps, d_out, interf);  // warm
            cudaMemcpyToSymbol(g_stop, &zero, 4);
            rate_kernel<<<148, 384, smem>>>(mode, n, reps, d_out, interf);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) {
                printf("mode %d n %d: %s\n", mode, n, cudaGetErrorString(e));
                return 1;
            }
            long long h[148];
            cudaMemcpy(h, d_out, sizeof h, cudaMemcpyDeviceToHost);
            double avg = 0;
            for (int i = 0; i < 148; ++i) avg += h[i];
            avg /= 148;
            const double per = avg / (reps * 8.0);
            printf("random %d interference %d mode %s N=%3d: %.1f cycles/UMMA  (%.0f flop/clk/SM)\n", rnd, interf, mode == 0 ? "SS" : "TS", n,
                   per, 2.0 * 128 * n * 16 / per);
        }
    }
    return 0;
}
