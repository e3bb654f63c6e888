// Probe of the tcgen05 building blocks the attention kernel relies on:
//   1. SS  MMA: D = A(K-major, smem, SW128) * B(K-major, smem, SW128)^T    (S = Q K^T)
//   2. TS  MMA: D = P(TMEM, packed bf16) * V(MN-major, smem, SW128)         (O = P V)
//   3. SS  MMA with MN-major B                                              (fallback for 2)
// Each result is checked against a host fp32 GEMM of the same bf16 inputs.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../../paper_2602_03216_b200/csrc/sm100.cuh"

using namespace tsa_dev;

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e = (x);                                                           \
        if (e != cudaSuccess) {                                                        \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            exit(1);                                                                   \
        }                                                                              \
    } while (0)

constexpr int M = 128, N = 128, K = 128;

struct __align__(1024) Smem {
    __nv_bfloat16 a[2][128 * 64];  // two 64-wide K blocks, SW128
    __nv_bfloat16 b[2][128 * 64];
    uint64_t bar_tma;
    uint64_t bar_mma;
    uint32_t tmem_base;
};

// mode 0: SS K-major/K-major; mode 1: TS with B MN-major; mode 2: SS A K-major, B MN-major
// mode 3: as 0, but B's 128 rows gathered by index from a larger matrix (TMA tile::gather4)
__global__ void probe_kernel(const __grid_constant__ CUtensorMap tmA,
                             const __grid_constant__ CUtensorMap tmB, const __nv_bfloat16* A_gl,
                             float* D, int mode, const __grid_constant__ CUtensorMap tmG,
                             const int* gidx) {
    extern __shared__ uint8_t raw[];
    Smem& s = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    const uint32_t warp = warp_id_uniform();
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
    const uint32_t tmem_d = tmem;          // cols [0,128)
    const uint32_t tmem_p = tmem + 128;    // cols [128,192): P packed bf16

    if (mode == 1) {
        // P (= A_gl, 128x128 row-major) into TMEM: thread t owns row t, packs (2c, 2c+1).
        const int row = threadIdx.x;
        const uint32_t lane_base = (warp * 32u) << 16;
        for (int c0 = 0; c0 < 64; c0 += 16) {
            uint32_t r[16];
            for (int j = 0; j < 16; ++j) {
                const __nv_bfloat16* p = A_gl + row * K + 2 * (c0 + j);
                __nv_bfloat162 v;
                v.x = p[0];
                v.y = p[1];
                r[j] = *reinterpret_cast<uint32_t*>(&v);
            }
            tmem_st16(tmem_p + lane_base + c0, r);
        }
        tmem_wait_st();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();

    if (threadIdx.x == 0) {
        uint32_t bytes = 0;
        if (mode != 1) {
            tma_load_2d(s.a[0], &tmA, &s.bar_tma, 0, 0);
            tma_load_2d(s.a[1], &tmA, &s.bar_tma, 64, 0);
            bytes += 2 * 128 * 64 * 2;
        }
        if (mode == 3) {
            for (int g = 0; g < 32; ++g) {
                const int* r = gidx + 4 * g;
                tma_gather4(reinterpret_cast<uint8_t*>(s.b[0]) + g * 512, &tmG, &s.bar_tma, 0, r[0], r[1], r[2], r[3]);
                tma_gather4(reinterpret_cast<uint8_t*>(s.b[1]) + g * 512, &tmG, &s.bar_tma, 64, r[0], r[1], r[2], r[3]);
            }
        } else {
            tma_load_2d(s.b[0], &tmB, &s.bar_tma, 0, 0);
            tma_load_2d(s.b[1], &tmB, &s.bar_tma, 64, 0);
        }
        bytes += 2 * 128 * 64 * 2;
        mbar_arrive_expect_tx(&s.bar_tma, bytes);
        mbar_wait(&s.bar_tma, 0);
        tc_fence_after();
        const uint32_t a0 = smem_u32(s.a[0]);
        const uint32_t b0 = smem_u32(s.b[0]);
        if (mode == 0 || mode == 3) {
            const uint32_t idesc = idesc_bf16_f32(M, N, 0, 0);
            for (int kk = 0; kk < K / 16; ++kk) {
                const uint32_t off = (kk / 4) * (128 * 128) + (kk % 4) * 32;
                mma_bf16_ss(tmem_d, sdesc_kmajor_sw128(a0 + off), sdesc_kmajor_sw128(b0 + off),
                            idesc, kk > 0);
            }
        } else {
            // B = V stored [K rows][N cols] (N contiguous): MN-major. Two 64-wide N blocks
            // 16 KiB apart; a K step of 16 rows advances 16 * 128 B = 2 KiB.
            const uint32_t idesc = idesc_bf16_f32(M, N, 0, 1);
            for (int kk = 0; kk < K / 16; ++kk) {
                const uint64_t bd = sdesc_mnmajor_sw128(b0 + kk * 2048, 128 * 128);
                if (mode == 1) {
                    mma_bf16_ts(tmem_d, tmem_p + kk * 8, bd, idesc, kk > 0);
                } else {
                    const uint32_t off = (kk / 4) * (128 * 128) + (kk % 4) * 32;
                    mma_bf16_ss(tmem_d, sdesc_kmajor_sw128(a0 + off), bd, idesc, kk > 0);
                }
            }
        }
        mma_commit(&s.bar_mma);
    }
    __syncwarp();
    mbar_wait(&s.bar_mma, 0);
    tc_fence_after();
    // epilogue: 4 warps, thread = row
    const int row = threadIdx.x;
    for (int c0 = 0; c0 < N; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(tmem_d + ((warp * 32u) << 16) + c0, r);
        tmem_wait_ld();
        for (int j = 0; j < 32; ++j) D[row * N + c0 + j] = __uint_as_float(r[j]);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 256);
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
}

static CUtensorMap make_map(void* base, int rows, int cols, int box_rows = 128) {
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = get_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box,
                              es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        printf("encode failed %d\n", (int)r);
        exit(1);
    }
    return m;
}

int main() {
    std::vector<__nv_bfloat16> hA(M * K), hB(N * K);
    std::vector<float> fA(M * K), fB(N * K);
    srand(1);
    for (int i = 0; i < M * K; ++i) {
        hA[i] = __float2bfloat16((rand() % 17 - 8) / 8.0f);
        fA[i] = __bfloat162float(hA[i]);
    }
    for (int i = 0; i < N * K; ++i) {
        hB[i] = __float2bfloat16((rand() % 13 - 6) / 4.0f);
        fB[i] = __bfloat162float(hB[i]);
    }
    __nv_bfloat16 *dA, *dB;
    float* dD;
    CK(cudaMalloc(&dA, M * K * 2));
    CK(cudaMalloc(&dB, N * K * 2));
    CK(cudaMalloc(&dD, M * N * 4));
    CK(cudaMemcpy(dA, hA.data(), M * K * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, hB.data(), N * K * 2, cudaMemcpyHostToDevice));
    CUtensorMap tA = make_map(dA, M, K), tB = make_map(dB, 128, 128);
    // gather source: 1000 rows; B = rows gidx[0..127] of it
    const int NG = 1000;
    std::vector<__nv_bfloat16> hG(NG * K);
    std::vector<float> fG(NG * K);
    for (int i = 0; i < NG * K; ++i) {
        hG[i] = __float2bfloat16((rand() % 11 - 5) / 4.0f);
        fG[i] = __bfloat162float(hG[i]);
    }
    std::vector<int> hidx(128);
    for (int i = 0; i < 128; ++i) hidx[i] = (i * 7919 + 13) % NG;
    __nv_bfloat16* dG;
    int* didx;
    CK(cudaMalloc(&dG, NG * K * 2));
    CK(cudaMalloc(&didx, 128 * 4));
    CK(cudaMemcpy(dG, hG.data(), NG * K * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(didx, hidx.data(), 128 * 4, cudaMemcpyHostToDevice));
    CUtensorMap tG = make_map(dG, NG, K, 1);
    const int smem = sizeof(Smem) + 1024;
    CK(cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int fails = 0;
    for (int mode = 0; mode < 4; ++mode) {
        CK(cudaMemset(dD, 0, M * N * 4));
        probe_kernel<<<1, 128, smem>>>(tA, tB, dA, dD, mode, tG, didx);
        CK(cudaDeviceSynchronize());
        std::vector<float> hD(M * N);
        CK(cudaMemcpy(hD.data(), dD, M * N * 4, cudaMemcpyDeviceToHost));
        double maxerr = 0;
        for (int i = 0; i < M; ++i)
            for (int j = 0; j < N; ++j) {
                double ref = 0;
                for (int k = 0; k < K; ++k) {
                    // mode 0: B is [N][K]; modes 1,2: B is V = [K][N]
                    const float b = mode == 0 ? fB[j * K + k]
                                    : mode == 3 ? fG[hidx[j] * K + k] : fB[k * N + j];
                    ref += (double)fA[i * K + k] * b;
                }
                maxerr = fmax(maxerr, fabs(ref - hD[i * N + j]));
            }
        printf("mode %d (%s): max_abs_err = %g  D[0][0]=%g D[5][77]=%g\n", mode,
               mode == 0 ? "SS kmajor" : mode == 1 ? "TS P-in-TMEM, V mn-major"
               : mode == 2 ? "SS V mn-major" : "SS, B rows by TMA gather4",
               maxerr, hD[0], hD[5 * N + 77]);
        if (maxerr > 1e-3) ++fails;
    }
    printf(fails ? "PROBE FAIL\n" : "PROBE OK\n");
    return fails;
}
