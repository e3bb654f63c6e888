// Peer memory for the fused multi-GPU exchanges: CUDA IPC buffers that every
// rank maps (over NVLink / NVSwitch between GPUs, or locally when ranks share
// a device), and a cross-rank barrier on the stream over IPC-mapped signal
// slots.  The producing kernels store score / output rows straight into the
// peers' buffers (OutReplicas); the barrier orders the consumers after them.
#include <cuda_runtime.h>

#include <cstdlib>
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

// Signal array of one barrier channel on one rank: int32 [world + 2] -- slots
// [0, world) receive the peers' arrivals, [world] is this rank's epoch counter
// (on the device, so a captured graph replays the barrier correctly: every
// rank runs the same barrier sequence, so the counters advance in lockstep),
// [world + 1] the timeout flag.
//
// Thread 0 advances the counter (host epoch < 1) or takes the host's epoch;
// thread r publishes this rank's arrival in rank r's slot [rank] (release at
// system scope, after a system fence so the data stores of the kernels before
// this one on the stream are visible first), then waits for rank r's arrival in
// this rank's slot [r] (acquire).  A peer that has not arrived after
// timeout_ns sets the timeout flag and returns (no trap: the context stays
// usable; the host checks the flag, tsa_peer_check).
__global__ void peer_barrier_kernel(SigPtrs s, int world, int rank, int epoch_host,
                                    unsigned long long timeout_ns) {
    __shared__ int epoch;
    int32_t* own = s.p[rank];
    if (threadIdx.x == 0) {
        epoch = epoch_host >= 1 ? epoch_host : own[world] + 1;
        own[world] = epoch;
    }
    __syncthreads();
    const int r = threadIdx.x;
    if (r >= world) return;
    __threadfence_system();
    asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(s.p[r] + rank), "r"(epoch) : "memory");
    const uint64_t t0 = global_ns();
    int v;
    do {
        asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(own + r) : "memory");
        if (v < epoch && global_ns() - t0 > timeout_ns) {
            atomicExch(own + world + 1, 1);
            return;
        }
    } while (v < epoch);
}

unsigned long long peer_timeout_ns() {
    static const unsigned long long ns = [] {
        const char* e = std::getenv("TSA_PEER_TIMEOUT_S");  // NCCL's default is 10 minutes
        const double sec = e ? std::atof(e) : 600.0;
        return (unsigned long long)((sec > 0 ? sec : 600.0) * 1e9);
    }();
    return ns;
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

namespace tsa {
int launch_peer_barrier(int32_t* const* signals, int world, int rank, cudaStream_t st) {
    SigPtrs s{};
    for (int r = 0; r < world; ++r) s.p[r] = signals[r];
    peer_barrier_kernel<<<1, 32, 0, st>>>(s, world, rank, 0, peer_timeout_ns());
    TSA_LAUNCH_CHECK("peer_barrier");
    return 0;
}
}  // namespace tsa

int tsa_peer_barrier(int32_t* const* signals, int32_t world, int32_t rank, int32_t epoch,
                     void* stream) {
    if (!signals || world < 1 || world > TSA_MAX_REPLICAS || rank < 0 || rank >= world)
        return invalid("tsa_peer_barrier: bad arguments (world " + std::to_string(world) +
                       ", rank " + std::to_string(rank) + ")");
    SigPtrs s{};
    for (int r = 0; r < world; ++r) {
        if (!signals[r]) return invalid("tsa_peer_barrier: null signal array");
        s.p[r] = signals[r];
    }
    peer_barrier_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(
        s, world, rank, epoch, peer_timeout_ns());
    TSA_LAUNCH_CHECK("peer_barrier");
    return 0;
}

int tsa_peer_check(const int32_t* own_signals, int32_t world, int32_t n_channels, void* stream) {
    if (!own_signals || world < 1 || world > TSA_MAX_REPLICAS || n_channels < 1)
        return invalid("tsa_peer_check: bad arguments");
    for (int c = 0; c < n_channels; ++c) {
        int32_t flag = 0;
        cudaError_t e = cudaMemcpyAsync(&flag, own_signals + c * (world + 2) + world + 1, 4,
                                        cudaMemcpyDeviceToHost, static_cast<cudaStream_t>(stream));
        if (e == cudaSuccess) e = cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
        if (e != cudaSuccess) return cuda_check(e, "tsa_peer_check");
        if (flag)
            return cuda_check(cudaErrorTimeout, ("tsa_peer_check: a peer did not reach barrier "
                                                 "channel " + std::to_string(c)).c_str());
    }
    return 0;
}
