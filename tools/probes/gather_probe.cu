// HBM probe for the K/V gather + zero-row pass (K4): the kernel's traffic is
// write-dominated (per 128K layer ~0.3 GB of reads, ~1.7 GB of writes), so its
// ceiling is the write bandwidth, not the copy bandwidth of MEASURED_PEAKS.
// Measures: copy (1:1), pure write, and gather-like variants on synthetic
// selections (rows per block, store cache hint).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_probe gather_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s\n", cudaGetErrorString(e)); return 1; } } while (0)

__global__ void fill_kernel(uint4* p, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        p[i] = make_uint4(0, 0, 0, 0);
}
__global__ void copy_kernel(const uint4* a, uint4* b, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        b[i] = a[i];
}

// ROWS rows of one head per block; 16 uint4 per row (d = 128 bf16).
template <int ROWS, bool CS>
__global__ void __launch_bounds__(256) gather_zero(const uint4* __restrict__ k, const uint4* __restrict__ v,
                                                   const int* __restrict__ idx, const int* __restrict__ inv,
                                                   int n, int L, int group, uint4* kc, uint4* vc, uint4* out) {
    __shared__ int rows[ROWS];
    __shared__ bool drop[ROWS];
    const int hg = blockIdx.x % group, rb = blockIdx.x / group;
    const int h = blockIdx.y * group + hg, kv = h / group;
    const int r0 = rb * ROWS;
    const int pad_end = min(L, (n + 127) / 128 * 128);
    const bool gather = r0 < pad_end;
    for (int i = threadIdx.x; i < ROWS; i += 256) {
        const int r = r0 + i;
        rows[i] = gather && r < n ? idx[(size_t)h * L + r] : -1;
        drop[i] = r < L && inv[(size_t)h * L + r] < 0;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < ROWS * 16; e += 256)
        if (drop[e / 16]) {
            if (CS) __stcs(out + ((size_t)h * L + r0) * 16 + e, make_uint4(0, 0, 0, 0));
            else out[((size_t)h * L + r0) * 16 + e] = make_uint4(0, 0, 0, 0);
        }
    if (!gather) return;
    constexpr int U = 4;
    for (int e0 = threadIdx.x; e0 < ROWS * 16; e0 += 256 * U) {
        uint4 kb[U], vb[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int e = e0 + u * 256;
            kb[u] = vb[u] = make_uint4(0, 0, 0, 0);
            if (e < ROWS * 16) {
                const int t = rows[e / 16];
                if (t >= 0) {
                    kb[u] = __ldg(k + ((size_t)kv * L + t) * 16 + e % 16);
                    vb[u] = __ldg(v + ((size_t)kv * L + t) * 16 + e % 16);
                }
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int e = e0 + u * 256;
            if (e >= ROWS * 16 || r0 + e / 16 >= pad_end) continue;
            const size_t dst = ((size_t)h * L + r0) * 16 + e;
            kc[dst] = kb[u];
            vc[dst] = vb[u];
        }
    }
}

template <int ROWS, bool CS>
float run(const uint4* k, const uint4* v, const int* idx, const int* inv, int n, int L, int H, int group,
          uint4* kc, uint4* vc, uint4* out) {
    dim3 grid((L + ROWS - 1) / ROWS * group, H / group);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int w = 0; w < 3; ++w) gather_zero<ROWS, CS><<<grid, 256>>>(k, v, idx, inv, n, L, group, kc, vc, out);
    cudaEventRecord(a);
    for (int it = 0; it < 20; ++it) gather_zero<ROWS, CS><<<grid, 256>>>(k, v, idx, inv, n, L, group, kc, vc, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    return ms / 20;
}

int main() {
    const int L = 131072, H = 32, HKV = 8, group = 4, n = 75533;
    const size_t row = 256, kvb = (size_t)HKV * L * row, hb = (size_t)H * L * row;
    uint4 *k, *v, *kc, *vc, *out;
    int *idx, *inv;
    CK(cudaMalloc(&k, kvb)); CK(cudaMalloc(&v, kvb)); CK(cudaMalloc(&kc, hb)); CK(cudaMalloc(&vc, hb));
    CK(cudaMalloc(&out, hb)); CK(cudaMalloc(&idx, (size_t)H * L * 4)); CK(cudaMalloc(&inv, (size_t)H * L * 4));
    // per head: n sorted distinct tokens (random), inverse map
    std::vector<int> hidx((size_t)H * L, 0), hinv((size_t)H * L, -1);
    std::mt19937 rng(1);
    std::vector<int> perm(L);
    for (int h = 0; h < H; ++h) {
        for (int i = 0; i < L; ++i) perm[i] = i;
        std::shuffle(perm.begin(), perm.end(), rng);
        std::sort(perm.begin(), perm.begin() + n);
        for (int r = 0; r < n; ++r) { hidx[(size_t)h * L + r] = perm[r]; hinv[(size_t)h * L + perm[r]] = r; }
    }
    CK(cudaMemcpy(idx, hidx.data(), hidx.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(inv, hinv.data(), hinv.size() * 4, cudaMemcpyHostToDevice));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    float ms;
    const size_t nwrite = hb / 16;
    for (int w = 0; w < 3; ++w) fill_kernel<<<148 * 8, 256>>>(out, nwrite);
    cudaEventRecord(a); for (int it = 0; it < 10; ++it) fill_kernel<<<148 * 8, 256>>>(out, nwrite); cudaEventRecord(b);
    cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b); ms /= 10;
    printf("write-only %.0f GB/s (%.2f GB in %.3f ms)\n", hb / ms / 1e6, hb / 1e9, ms);
    const size_t ncopy = hb / 2 / 16;
    for (int w = 0; w < 3; ++w) copy_kernel<<<148 * 8, 256>>>(kc, vc, ncopy);
    cudaEventRecord(a); for (int it = 0; it < 10; ++it) copy_kernel<<<148 * 8, 256>>>(kc, vc, ncopy); cudaEventRecord(b);
    cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b); ms /= 10;
    printf("copy (r+w) %.0f GB/s\n", 2.0 * ncopy * 16 / ms / 1e6);
    // algorithmic bytes of the gather + zero pass (bench.py's formula)
    const double alg = 4.0 * H * n * row + 4.0 * H * n + (double)H * (L - n) * row + 4.0 * H * L;
    float t;
    t = run<64, false>(k, v, idx, inv, n, L, H, group, kc, vc, out);  printf("gather rows=64          %.3f ms  %.0f GB/s alg\n", t, alg / t / 1e6);
    t = run<64, true>(k, v, idx, inv, n, L, H, group, kc, vc, out);   printf("gather rows=64  zero.cs %.3f ms  %.0f GB/s alg\n", t, alg / t / 1e6);
    t = run<128, false>(k, v, idx, inv, n, L, H, group, kc, vc, out); printf("gather rows=128         %.3f ms  %.0f GB/s alg\n", t, alg / t / 1e6);
    t = run<256, false>(k, v, idx, inv, n, L, H, group, kc, vc, out); printf("gather rows=256         %.3f ms  %.0f GB/s alg\n", t, alg / t / 1e6);
    t = run<256, true>(k, v, idx, inv, n, L, H, group, kc, vc, out);  printf("gather rows=256 zero.cs %.3f ms  %.0f GB/s alg\n", t, alg / t / 1e6);
    return 0;
}
