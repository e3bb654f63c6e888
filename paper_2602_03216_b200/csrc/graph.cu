// CUDA-graph replay of the layer chain.
//
// The sparse-layer chain (score -> budget -> select -> gather -> attend) never
// synchronises with the host: k_keep stays in device memory and every kernel
// sizes its grid for L and reads n from there.  Its launch sequence is
// therefore a pure function of the descriptor and the buffer addresses, so it
// is captured once per (descriptor, pointers) key and replayed with one
// cudaGraphLaunch -- removing the host launch gaps between the short
// selection kernels (~0.5 ms per 128K layer measured eagerly).
//
// Capture runs on a private non-blocking stream in relaxed mode, so the
// caller's stream may be the legacy default stream.  A call on a stream that
// is itself being captured (a caller-level graph) runs eagerly into that
// capture.  TSA_GRAPHS=0 disables replay.
#include <cstdlib>
#include <cstring>
#include <list>
#include <mutex>

#include "common.cuh"

namespace tsa {

namespace {

struct Key {
    tsa_desc d;
    const void* p[kGraphPtrs];
    int device;
};

bool same(const Key& a, const Key& b) { return std::memcmp(&a, &b, sizeof(Key)) == 0; }

struct Entry {
    Key key;
    cudaGraphExec_t exec;
    unsigned long long launches;  // kernels in the graph (tsa_kernel_launches)
};

constexpr size_t kMaxEntries = 16;

std::mutex g_mu;
std::list<Entry> g_cache;  // most recent first

bool graphs_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("TSA_GRAPHS");
        return !(e && e[0] == '0');
    }();
    return on;
}

cudaStream_t capture_stream(int device) {
    static thread_local cudaStream_t s[64] = {};
    if (device < 0 || device >= 64) return nullptr;
    if (!s[device] && cudaStreamCreateWithFlags(&s[device], cudaStreamNonBlocking) != cudaSuccess)
        return nullptr;
    return s[device];
}

}  // namespace

int graph_launch(const tsa_desc& d, const std::array<const void*, kGraphPtrs>& ptrs,
                 cudaStream_t st, const std::function<int(cudaStream_t)>& body) {
    if (!graphs_enabled()) return body(st);
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
        cudaGetLastError();
        return body(st);
    }
    Key key;
    std::memset(&key, 0, sizeof key);  // padding bytes take part in the comparison
    key.d = d;
    for (int i = 0; i < kGraphPtrs; ++i) key.p[i] = ptrs[i];
    if (cudaGetDevice(&key.device) != cudaSuccess) return cuda_check(cudaGetLastError(), "graph");

    std::lock_guard<std::mutex> lock(g_mu);
    for (auto it = g_cache.begin(); it != g_cache.end(); ++it) {
        if (!same(it->key, key)) continue;
        if (it != g_cache.begin()) g_cache.splice(g_cache.begin(), g_cache, it);
        cudaError_t e = cudaGraphLaunch(g_cache.front().exec, st);
        if (e != cudaSuccess) return cuda_check(e, "cudaGraphLaunch");
        add_launches(g_cache.front().launches);
        return 0;
    }
    cudaStream_t cap = capture_stream(key.device);
    if (!cap) return body(st);
    const unsigned long long before = launches_so_far();
    if (cudaStreamBeginCapture(cap, cudaStreamCaptureModeRelaxed) != cudaSuccess) {
        cudaGetLastError();
        return body(st);
    }
    const int rc = body(cap);
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(cap, &graph);
    const unsigned long long n = launches_so_far() - before;
    add_launches(0ull - n);  // captured, not executed
    if (rc != 0) {  // a validation error: report it, as the eager call would
        if (graph) cudaGraphDestroy(graph);
        return rc;
    }
    cudaGraphExec_t exec = nullptr;
    if (e == cudaSuccess) e = cudaGraphInstantiate(&exec, graph, 0);
    if (graph) cudaGraphDestroy(graph);
    if (e != cudaSuccess) {  // not capturable here (e.g. pageable k_keep_host): run eagerly
        cudaGetLastError();
        return body(st);
    }
    if (g_cache.size() >= kMaxEntries) {
        cudaGraphExecDestroy(g_cache.back().exec);
        g_cache.pop_back();
    }
    g_cache.push_front(Entry{key, exec, n});
    e = cudaGraphLaunch(exec, st);
    if (e != cudaSuccess) return cuda_check(e, "cudaGraphLaunch");
    add_launches(n);
    return 0;
}

void graph_cache_clear() {
    std::lock_guard<std::mutex> lock(g_mu);
    for (auto& en : g_cache) cudaGraphExecDestroy(en.exec);
    g_cache.clear();
}

}  // namespace tsa
