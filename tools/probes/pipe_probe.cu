// Per-SM issue / pipe throughput of the instructions the attention softmax is
// made of (diagnostic): MUFU ex2, bf16x2 pack, packed f32x2 FMA/ADD, 3-input
// max, round-down add.  Prints warp-instructions per clock per SM for each op
// alone and for pairs (to see which ops share a pipe).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_probe pipe_probe.cu
#include <cstdint>
#include <cstdio>

#define CH 8
#define ITERS 4096

__device__ __forceinline__ float op_ex2(float x) {
    float y;
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float op_cvt(float x, float y) {
    uint32_t r;
    asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(x), "f"(y));
    return __uint_as_float(r);
}
__device__ __forceinline__ float op_fma(float x) {
    float y;
    asm volatile("fma.rn.f32 %0, %1, 0f3F800001, 0f3A000000;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float op_addrm(float x) {
    float y;
    asm volatile("add.rm.f32 %0, %1, 0f4B400000;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float op_max3(float x, float a, float b) {
    float y;
    asm volatile("max.f32 %0, %1, %2, %3;" : "=f"(y) : "f"(x), "f"(a), "f"(b));
    return y;
}
__device__ __forceinline__ float op_max(float x, float a) {
    float y;
    asm volatile("max.f32 %0, %1, %2;" : "=f"(y) : "f"(x), "f"(a));
    return y;
}
__device__ __forceinline__ float op_imad(float x) {
    uint32_t y;
    asm volatile("mad.lo.u32 %0, %1, 8388608, 7;" : "=r"(y) : "r"(__float_as_uint(x)));
    return __uint_as_float(y);
}
__device__ __forceinline__ void op_fma2(float& x0, float& x1) {
    uint64_t v = ((uint64_t)__float_as_uint(x1) << 32) | __float_as_uint(x0), r;
    const uint64_t a = 0x3F8000013F800001ull, c = 0x3A0000003A000000ull;
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(v), "l"(a), "l"(c));
    x0 = __uint_as_float((uint32_t)r);
    x1 = __uint_as_float((uint32_t)(r >> 32));
}
__device__ __forceinline__ void op_add2(float& x0, float& x1) {
    uint64_t v = ((uint64_t)__float_as_uint(x1) << 32) | __float_as_uint(x0), r;
    const uint64_t c = 0x3A0000003A000000ull;
    asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(v), "l"(c));
    x0 = __uint_as_float((uint32_t)r);
    x1 = __uint_as_float((uint32_t)(r >> 32));
}

// packed exponentials: two results per lane per instruction
__device__ __forceinline__ float op_ex2_h2(float x) {
    uint32_t y;
    asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(__float_as_uint(x)));
    return __uint_as_float(y);
}
__device__ __forceinline__ float op_ex2_bf2(float x) {
    uint32_t y;
    asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(__float_as_uint(x)));
    return __uint_as_float(y);
}
__device__ __forceinline__ float op_cvt_h2(float x, float y) {
    uint32_t r;
    asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(x), "f"(y));
    return __uint_as_float(r);
}

template <int OP>
__global__ void probe(float* out, long long* cyc, float seed) {
    float x[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = seed * (threadIdx.x + i) * 1e-9f - 0.5f;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) {
            if (OP == 0) x[i] = op_ex2(x[i]);
            if (OP == 1) x[i] = op_cvt(x[i], x[(i + 1) % CH]);
            if (OP == 2) x[i] = op_fma(x[i]);
            if (OP == 3 && (i & 1) == 0) op_fma2(x[i], x[i + 1]);
            if (OP == 4) x[i] = op_addrm(x[i]);
            if (OP == 5) x[i] = op_max3(x[i], x[(i + 3) % CH], x[(i + 5) % CH]);
            if (OP == 6) x[i] = op_max(x[i], x[(i + 3) % CH]);
            if (OP == 7) x[i] = op_imad(x[i]);
            if (OP == 8 && (i & 1) == 0) op_add2(x[i], x[i + 1]);
            // pairs: ex2 + cvt, ex2 + fma2, ex2 + max3, cvt + fma2
            if (OP == 10) { x[i] = op_ex2(x[i]); x[i] = op_cvt(x[i], x[(i + 1) % CH]); }
            if (OP == 11) { x[i] = op_ex2(x[i]); if ((i & 1) == 0) op_fma2(x[i], x[i + 1]); }
            if (OP == 12) { x[i] = op_ex2(x[i]); x[i] = op_max3(x[i], x[(i + 3) % CH], x[(i + 5) % CH]); }
            if (OP == 13) { x[i] = op_cvt(x[i], x[(i + 1) % CH]); if ((i & 1) == 0) op_fma2(x[i], x[i + 1]); }
            if (OP == 14) { x[i] = op_ex2(x[i]); x[i] = op_imad(x[i]); }
            if (OP == 20) x[i] = op_ex2_h2(x[i]);
            if (OP == 21) x[i] = op_ex2_bf2(x[i]);
            if (OP == 22) x[i] = op_cvt_h2(x[i], x[(i + 1) % CH]);
            if (OP == 23) { x[i] = op_cvt_h2(x[i], x[(i + 1) % CH]); x[i] = op_ex2_h2(x[i]); }
        }
    }
    long long t1 = clock64();
    float s = 0;
#pragma unroll
    for (int i = 0; i < CH; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, double instr_per_elem, float* out, long long* cyc, int threads) {
    probe<OP><<<148, threads>>>(out, cyc, 1.0f);
    cudaDeviceSynchronize();
    probe<OP><<<148, threads>>>(out, cyc, 1.0f);
    cudaDeviceSynchronize();
    long long c[148];
    cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int i = 0; i < 148; ++i) mx = c[i] > mx ? c[i] : mx;
    const double warp_instr = (double)(threads / 32) * ITERS * CH * instr_per_elem;
    printf("%-22s threads=%4d  %.3f warp-instr/clk/SM  (%.1f lanes/clk/SM)\n", name, threads,
           warp_instr / mx, 32.0 * warp_instr / mx);
}

int main() {
    float* out;
    long long* cyc;
    cudaMalloc(&out, 148 * 1024 * 4);
    cudaMalloc(&cyc, 148 * 8);
    for (int th : {128, 512}) {
        run<0>("ex2.approx.ftz.f32", 1, out, cyc, th);
        run<1>("cvt.rn.bf16x2.f32", 1, out, cyc, th);
        run<2>("fma.rn.f32", 1, out, cyc, th);
        run<3>("fma.rn.f32x2", 0.5, out, cyc, th);
        run<8>("add.rn.f32x2", 0.5, out, cyc, th);
        run<4>("add.rm.f32", 1, out, cyc, th);
        run<5>("max.f32 (3 inputs)", 1, out, cyc, th);
        run<6>("max.f32", 1, out, cyc, th);
        run<7>("mad.lo.u32", 1, out, cyc, th);
        run<10>("ex2 + cvt (2 instr)", 2, out, cyc, th);
        run<11>("ex2 + fma2 (1.5)", 1.5, out, cyc, th);
        run<12>("ex2 + max3 (2)", 2, out, cyc, th);
        run<13>("cvt + fma2 (1.5)", 1.5, out, cyc, th);
        run<14>("ex2 + imad (2)", 2, out, cyc, th);
        run<20>("ex2.approx.f16x2", 1, out, cyc, th);
        run<21>("ex2.approx.ftz.bf16x2", 1, out, cyc, th);
        run<22>("cvt.rn.f16x2.f32", 1, out, cyc, th);
        run<23>("cvt f16x2 + ex2 f16x2", 2, out, cyc, th);
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
