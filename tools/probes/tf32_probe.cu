// Probe of the kind::tf32 building blocks attend_tf32.cu relies on:
//   mode 0  SS MMA: D = A(K-major, SW128 f32) * B(K-major, SW128 f32)^T, K = 32 (4 x K8)
//   mode 1  TS MMA: D = P(TMEM, f32 one per column) * V(MN-major, SW128 f32), K = 32 keys
//           V [32 keys x 128] loaded as 4 boxes {32 cols, 32 rows} 4 KiB apart
//   mode 2  SS MMA: D = P(K-major smem) * V(MN-major)
//   mode 3  TS MMA: D = P(TMEM) * Vt(K-major smem, V transposed on the host)
// Measured on B200: K-major SW128 works as for bf16; MN-major TF32 needs the
// 128-B swizzle with 32-B atoms (TMA CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
// descriptor layout 1 = SWIZZLE_128B_BASE32B) with SBO = 512 B (4-row K
// groups); plain SWIZZLE_128B reads as zeros, SBO = 1 KiB is wrong.
// Results vs a host double GEMM of the TF32-truncated inputs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 tf32_probe.cu -o /tmp/tf32_probe -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../../paper_2602_03216_b200/csrc/sm100.cuh"

using namespace tsa_dev;

#define CK(x)                                                                                \
    do {                                                                                     \
        cudaError_t e = (x);                                                                 \
        if (e != cudaSuccess) {                                                              \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);   \
            exit(1);                                                                         \
        }                                                                                    \
    } while (0)

struct __align__(1024) Smem {
    uint8_t a[16384];
    uint8_t b[16384];
    uint64_t bar_tma, bar_mma;
    uint32_t tmem_base;
};

__host__ __device__ constexpr uint32_t idesc_tf32(uint32_t b_mn) {
    return (1u << 4) | (2u << 7) | (2u << 10) | (b_mn << 16) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
}
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo) {
    return (static_cast<uint64_t>(0x40004040u) << 32) | (((saddr >> 4) & 0x3FFFu) | ((lbo >> 4) << 16));
}
// MN-major, SWIZZLE_128B_BASE32B (layout 1): 128-B rows, 32-B swizzle atoms
__device__ __forceinline__ uint64_t desc32(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    const uint32_t hi = (1u << 29) | (1u << 14) | ((sbo >> 4) & 0x3FFFu);
    return (static_cast<uint64_t>(hi) << 32) | (((saddr >> 4) & 0x3FFFu) | ((lbo >> 4) << 16));
}

__global__ void probe(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      const float* P, float* D, int mode, uint32_t SBO) {
    extern __shared__ uint8_t raw[];
    Smem& s = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    const uint32_t warp = warp_id_uniform(), lane = lane_id();
    if (threadIdx.x == 0) {
        mbar_init(&s.bar_tma, 1);
        mbar_init(&s.bar_mma, 1);
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc(&s.tmem_base, 256);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s.tmem_base;
    const uint32_t lane_off = (warp * 32) << 16;
    if (threadIdx.x == 0) {
        if (mode == 0 || mode == 3 || mode == 2) {
            mbar_arrive_expect_tx(&s.bar_tma, 2 * 16384);
            tma_load_2d(s.a, &tmA, &s.bar_tma, 0, 0);
            if (mode == 2) {
                for (int a = 0; a < 4; ++a) tma_load_2d(s.b + a * 4096, &tmB, &s.bar_tma, 32 * a, 0);
            } else {
                tma_load_2d(s.b, &tmB, &s.bar_tma, 0, 0);
            }
        } else {
            mbar_arrive_expect_tx(&s.bar_tma, 16384);
            for (int a = 0; a < 4; ++a) tma_load_2d(s.b + a * 4096, &tmB, &s.bar_tma, 32 * a, 0);
        }
    }
    if (mode == 1 || mode == 3) {  // P row (32 f32) of this thread's lane into TMEM cols [128, 160)
        uint32_t r[32];
        for (int e = 0; e < 32; ++e) r[e] = __float_as_uint(P[(warp * 32 + lane) * 32 + e]);
        tmem_st32(tmem + 128 + lane_off, r);
        tmem_wait_st();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x == 0) {
        mbar_wait(&s.bar_tma, 0);
        tc_fence_after();
        for (int kk = 0; kk < 4; ++kk) {
            if (mode == 0 || mode == 2) {
                const uint64_t bd = mode == 0 ? desc(smem_u32(s.b) + kk * 32, 16)
                                              : desc32(smem_u32(s.b) + kk * 1024, 4096, SBO);
                asm volatile(
                    "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                    "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                    "l"(desc(smem_u32(s.a) + kk * 32, 16)), "l"(bd),
                    "r"(idesc_tf32(mode == 2 ? 1 : 0)), "r"(kk));
            } else {
                asm volatile(
                    "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                    "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem),
                    "r"(tmem + 128 + kk * 8),
                    "l"(mode == 1 ? desc32(smem_u32(s.b) + kk * 1024, 4096, SBO) : desc(smem_u32(s.b) + kk * 32, 16)),
                    "r"(idesc_tf32(mode == 1 ? 1 : 0)), "r"(kk));
            }
        }
        mma_commit(&s.bar_mma);
    }
    __syncwarp();
    mbar_wait(&s.bar_mma, 0);
    tc_fence_after();
    for (int c = 0; c < 4; ++c) {
        uint32_t r[32];
        tmem_ld32(tmem + lane_off + c * 32, r);
        tmem_wait_ld();
        for (int e = 0; e < 32; ++e) D[(warp * 32 + lane) * 128 + c * 32 + e] = __uint_as_float(r[e]);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 256);
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}
static void map2d(CUtensorMap* m, const float* base, uint64_t inner, uint64_t rows, uint32_t bi,
                  uint32_t br, CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B) {
    cuuint64_t dims[2] = {inner, rows};
    cuuint64_t strides[1] = {inner * 4};
    cuuint32_t box[2] = {bi, br};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box,
                       es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        printf("encode failed %d\n", (int)r);
        exit(1);
    }
}
static float t32(float x) {
    uint32_t u;
    memcpy(&u, &x, 4);
    u &= 0xFFFFE000u;
    memcpy(&x, &u, 4);
    return x;
}

int main() {
    srand(1);
    auto rnd = [] { return (float)rand() / RAND_MAX * 2.0f - 1.0f; };
    std::vector<float> A(128 * 32), B(128 * 32), P(128 * 32), V(32 * 128), D(128 * 128), Vt(128 * 32);
    for (auto& x : A) x = rnd();
    for (auto& x : B) x = rnd();
    for (auto& x : P) x = rnd();
    for (auto& x : V) x = rnd();
    for (int k = 0; k < 32; ++k)
        for (int j = 0; j < 128; ++j) Vt[j * 32 + k] = V[k * 128 + j];
    float *dA, *dB, *dP, *dV, *dD, *dVt;
    CK(cudaMalloc(&dVt, Vt.size() * 4));
    CK(cudaMemcpy(dVt, Vt.data(), Vt.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMalloc(&dA, A.size() * 4));
    CK(cudaMalloc(&dB, B.size() * 4));
    CK(cudaMalloc(&dP, P.size() * 4));
    CK(cudaMalloc(&dV, V.size() * 4));
    CK(cudaMalloc(&dD, D.size() * 4));
    CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dP, P.data(), P.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dV, V.data(), V.size() * 4, cudaMemcpyHostToDevice));
    CUtensorMap mA, mB, mV, mP, mVt;
    map2d(&mP, dP, 32, 128, 32, 128);
    map2d(&mVt, dVt, 32, 128, 32, 128);
    map2d(&mA, dA, 32, 128, 32, 128);
    map2d(&mB, dB, 32, 128, 32, 128);
    map2d(&mV, dV, 128, 32, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    const int smem = sizeof(Smem) + 1024;
    CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    for (int cfg = 0; cfg < 6; ++cfg) {
        const int mode = cfg < 4 ? cfg : cfg - 3;
        const uint32_t SBO = cfg < 4 ? 512 : 1024;
        CK(cudaMemset(dD, 0, D.size() * 4));
        probe<<<1, 128, smem>>>(mode == 2 ? mP : mA, mode == 0 ? mB : mode == 3 ? mVt : mV, dP, dD, mode, SBO);
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
        double maxerr = 0, maxref = 0;
        int bad_i = -1, bad_j = -1;
        for (int i = 0; i < 128; ++i)
            for (int j = 0; j < 128; ++j) {
                double ref = 0;
                for (int k = 0; k < 32; ++k)
                    ref += mode == 0 ? (double)t32(A[i * 32 + k]) * t32(B[j * 32 + k])
                         : mode == 3 ? (double)t32(P[i * 32 + k]) * t32(Vt[j * 32 + k])
                                     : (double)t32(P[i * 32 + k]) * t32(V[k * 128 + j]);
                const double err = fabs(ref - D[i * 128 + j]);
                if (err > maxerr) maxerr = err, bad_i = i, bad_j = j;
                maxref = fmax(maxref, fabs(ref));
            }
        printf("SBO %u mode %d (%s): max |err| %.3e (max |ref| %.3e) at (%d, %d): got %g\n", SBO,
               mode, mode == 0 ? "SS K-major" : mode == 1 ? "TS, B MN-major" : mode == 2 ? "SS, B MN-major" : "TS, B K-major", maxerr, maxref, bad_i, bad_j,
               D[bad_i * 128 + bad_j]);
    }
    return 0;
}
