// Peer memory for the fused multi-GPU exchanges: CUDA IPC buffers that every
// rank maps (over NVLink / NVSwitch between GPUs, or locally when ranks share
// a device), and a cross-rank barrier on the stream over IPC-mapped signal
// slots.  The producing kernels store score / output rows straight into the
// peers' buffers (OutReplicas); the barrier orders the consumers after them.
#include <cuda_runtime.h>

#include <cstring>

#include "common.cuh"

namespace tsa {
namespace {

struct SigPtrs {
    int32_t* p[TSA_MAX_REPLICAS];
};

__device__ __forceinline__ uint64_t global_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Thread r: publish this rank's arrival in rank r's slot [rank] (release at
// system scope, after a system fence so the data stores of the kernels before
// this one on the stream are visible first), then wait for rank r's arrival
// in this rank's slot [r] (acquire).  A peer that never arrives traps after
// 60 s instead of hanging the GPU.
__global__ void peer_barrier_kernel(SigPtrs s, int world, int rank, int epoch) {
    const int r = threadIdx.x;
    if (r >= world) return;
    __threadfence_system();
    asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(s.p[r] + rank), "r"(epoch) : "memory");
    const uint64_t t0 = global_ns();
    int v;
    do {
        asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(s.p[rank] + r) : "memory");
        if (v < epoch && global_ns() - t0 > 60ull * 1000000000ull) __trap();
    } while (v < epoch);
}

}  // namespace
}  // namespace tsa

using namespace tsa;

int tsa_ipc_alloc(size_t bytes, void** ptr, void* handle) {
    if (!ptr || !handle || bytes == 0) return invalid("tsa_ipc_alloc: null pointer or zero size");
    cudaError_t e = cudaMalloc(ptr, bytes);
    if (e != cudaSuccess) return cuda_check(e, "tsa_ipc_alloc: cudaMalloc");
    if ((e = cudaMemset(*ptr, 0, bytes)) != cudaSuccess) return cuda_check(e, "tsa_ipc_alloc");
    cudaIpcMemHandle_t h;
    if ((e = cudaIpcGetMemHandle(&h, *ptr)) != cudaSuccess)
        return cuda_check(e, "tsa_ipc_alloc: cudaIpcGetMemHandle");
    static_assert(sizeof(h) == TSA_IPC_HANDLE_BYTES, "cudaIpcMemHandle_t size");
    std::memcpy(handle, &h, sizeof h);
    return 0;
}

int tsa_ipc_open(const void* handle, void** ptr) {
    if (!ptr || !handle) return invalid("tsa_ipc_open: null pointer");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof h);
    cudaError_t e = cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess);
    return e == cudaSuccess ? 0 : cuda_check(e, "tsa_ipc_open: cudaIpcOpenMemHandle");
}

int tsa_ipc_close(void* ptr) {
    cudaError_t e = cudaIpcCloseMemHandle(ptr);
    return e == cudaSuccess ? 0 : cuda_check(e, "tsa_ipc_close");
}

int tsa_ipc_free(void* ptr) {
    cudaError_t e = cudaFree(ptr);
    return e == cudaSuccess ? 0 : cuda_check(e, "tsa_ipc_free");
}

int tsa_peer_barrier(int32_t* const* signals, int32_t world, int32_t rank, int32_t epoch,
                     void* stream) {
    if (!signals || world < 1 || world > TSA_MAX_REPLICAS || rank < 0 || rank >= world ||
        epoch < 1)
        return invalid("tsa_peer_barrier: bad arguments (world " + std::to_string(world) +
                       ", rank " + std::to_string(rank) + ", epoch " + std::to_string(epoch) + ")");
    SigPtrs s{};
    for (int r = 0; r < world; ++r) {
        if (!signals[r]) return invalid("tsa_peer_barrier: null signal array");
        s.p[r] = signals[r];
    }
    peer_barrier_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(s, world, rank, epoch);
    TSA_LAUNCH_CHECK("peer_barrier");
    return 0;
}
