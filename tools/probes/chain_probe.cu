// Cycle cost of a sequential f32 FADD chain fed from shared memory (the
// exact scorer's row-sum chain): one warp, lane = row, 256 values per tile.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 chain_probe.cu -o chain_probe
#include <cstdio>
#include <cuda_runtime.h>

constexpr int KEYS = 256, EP = 17;

template <int MODE>
__global__ void chain(float* out, long long* cyc, int tiles) {
    __shared__ float e[KEYS * EP];
    for (int i = threadIdx.x; i < KEYS * EP; i += blockDim.x) e[i] = 1e-3f * (i % 7);
    __syncthreads();
    const int row = threadIdx.x & 15;
    float s = 0.f;
    long long t0 = clock64();
    for (int t = 0; t < tiles; ++t) {
        const float* es = e + row;
        if (MODE == 0) {
#pragma unroll
            for (int j = 0; j < KEYS; ++j) s = __fadd_rn(s, es[j * EP]);
        } else if (MODE == 1) {
            float v[KEYS];
#pragma unroll
            for (int j = 0; j < KEYS; ++j) v[j] = es[j * EP];
#pragma unroll
            for (int j = 0; j < KEYS; ++j) s = __fadd_rn(s, v[j]);
        } else {  // pure chain on registers (lower bound)
#pragma unroll
            for (int j = 0; j < KEYS; ++j) s = __fadd_rn(s, __int_as_float(j + t));
        }
        __syncwarp();
    }
    long long t1 = clock64();
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[MODE] = t1 - t0;
}

int main() {
    float* out;
    long long* cyc;
    cudaMalloc(&out, 1024);
    cudaMallocManaged(&cyc, 64);
    const int tiles = 512;
    chain<0><<<1, 32>>>(out, cyc, tiles);
    chain<1><<<1, 32>>>(out, cyc, tiles);
    chain<2><<<1, 32>>>(out, cyc, tiles);
    cudaDeviceSynchronize();
    for (int m = 0; m < 3; ++m)
        printf("mode %d: %.2f cycles per element\n", m, (double)cyc[m] / (tiles * KEYS));
    return 0;
}
