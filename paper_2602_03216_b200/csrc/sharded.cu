// The head-sharded layer as one C-ABI call (tsa_sparse_attention_layer_sharded):
// the caller side of model.cpp:169-183 when the heads of a layer are split over
// G GPUs, one process per GPU.  Rank g owns query heads
// [head_begin, head_end) and their KV heads; score, select, compress, attend and
// decompress are local, and the two exchanges run in one of two forms:
//
//  peer  (tsa_peer): the score rows and the output rows are stored by the
//        producing kernels straight into every rank's buffer (CUDA IPC over
//        NVLink); device-side barriers (epoch counters in device memory, so the
//        call can be captured in a CUDA graph and replayed) order the budget
//        after the scores and end the step;
//  nccl  (ncclComm_t): ncclAllGather of the score rows before the budget and
//        of the output rows after the attention, in place.
//
// NCCL is resolved at run time (dlopen of libnccl.so.2, normally the one the
// process already loaded), so the library has no link-time NCCL dependency.
#include <dlfcn.h>

#include <mutex>
#include <string>

#include "common.cuh"

namespace tsa {
namespace {

// ncclResult_t ncclAllGather(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t)
using AllGatherFn = int (*)(const void*, void*, size_t, int, void*, cudaStream_t);
using ErrorStringFn = const char* (*)(int);
constexpr int kNcclFloat32 = 7, kNcclBfloat16 = 9;  // nccl.h ncclDataType_t

struct Nccl {
    AllGatherFn all_gather = nullptr;
    ErrorStringFn error_string = nullptr;
};

const Nccl* nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the process's NCCL
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        n.all_gather = reinterpret_cast<AllGatherFn>(dlsym(h, "ncclAllGather"));
        n.error_string = reinterpret_cast<ErrorStringFn>(dlsym(h, "ncclGetErrorString"));
    });
    return n.all_gather ? &n : nullptr;
}

int nccl_check(int r, const char* what) {
    if (r == 0) return 0;
    const Nccl* n = nccl();
    set_error(std::string(what) + ": " +
              (n && n->error_string ? n->error_string(r) : ("NCCL error " + std::to_string(r))));
    return TSA_ERR_NCCL;
}

OutReplicas replicas(void* const* bases, int world, size_t offset_bytes) {
    OutReplicas r{};
    for (int i = 0; i < world; ++i) r.p[i] = static_cast<uint8_t*>(bases[i]) + offset_bytes;
    r.n = world;
    return r;
}

}  // namespace
}  // namespace tsa

using namespace tsa;

int tsa_sparse_attention_layer_sharded(const tsa_desc* d, const void* q, const void* k,
                                       const void* v, const tsa_peer* peer, void* nccl_comm,
                                       float* s_full, void* out_full, int32_t* k_keep, void* ws,
                                       void* stream) {
    if (int rc = check_descriptor(d)) return rc;
    if (!q || !k || !v || !k_keep || !ws)
        return invalid("tsa_sparse_attention_layer_sharded: null buffer");
    if ((peer == nullptr) == (nccl_comm == nullptr))
        return invalid("tsa_sparse_attention_layer_sharded: exactly one of peer and nccl_comm");
    const int H = d->n_heads, Hkv = d->n_kv_heads, g = H / Hkv;
    const int h0 = d->head_begin, h1 = d->head_end, nh = h1 - h0;
    const size_t L = d->seq_len, D = d->d_head, eb = elem_bytes(d->dtype);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // the shard as a self-contained layer (heads numbered from 0, as the
    // per-rank descriptors of dist.py), and the whole layer for the budget
    tsa_desc dl = *d;
    dl.n_heads = nh;
    dl.n_kv_heads = nh / g;
    dl.head_begin = 0;
    dl.head_end = nh;
    tsa_desc df = *d;
    df.head_begin = 0;
    df.head_end = H;
    const Workspace w = workspace_layout(dl);
    auto at_ws = [&](size_t off) { return static_cast<uint8_t*>(ws) + off; };
    int32_t* idx = reinterpret_cast<int32_t*>(at_ws(w.idx));
    int32_t* inv = reinterpret_cast<int32_t*>(at_ws(w.inv));
    const int fb = forced_begin_of(*d), nf = d->seq_len - fb;
    const bool dense = d->mode == TSA_MODE_DENSE;
    int rc;
    if (peer) {
        const int world = peer->world, rank = peer->rank;
        if (world < 1 || world > TSA_MAX_REPLICAS || rank < 0 || rank >= world)
            return invalid("tsa_sparse_attention_layer_sharded: bad peer world / rank");
        if (!attend_sm100_supported(*d))
            return invalid("tsa_sparse_attention_layer_sharded: the peer form needs the fused "
                           "bf16 / d_head 128 path");
        for (int r = 0; r < world; ++r)
            if (!peer->scores[r] || !peer->out[r] || !peer->signals[0][r] ||
                !peer->signals[1][r] || !peer->signals[2][r])
                return invalid("tsa_sparse_attention_layer_sharded: null peer buffer");
        const OutReplicas out_rep = replicas(peer->out, world, (size_t)h0 * L * D * eb);
        // no rank overwrites a buffer a peer may still read (the previous step)
        if ((rc = launch_peer_barrier(peer->signals[0], world, rank, st))) return rc;
        if (dense) {
            if ((rc = launch_write_int(k_keep, d->seq_len, st))) return rc;
            if ((rc = launch_attend_sm100_rep(dl, q, k, v, out_rep, st))) return rc;
            return launch_peer_barrier(peer->signals[1], world, rank, st);
        }
        // C1 fused into the pool pass: this shard's score rows to every rank
        const OutReplicas s_rep =
            replicas(reinterpret_cast<void* const*>(peer->scores), world, (size_t)h0 * L * 4);
        if ((rc = score_stage(dl, q, k, s_rep, ws, st))) return rc;
        if ((rc = launch_peer_barrier(peer->signals[2], world, rank, st))) return rc;
        float* s_all = peer->scores[rank];
        if ((rc = budget_stage(df, s_all, k_keep, ws, std::max(1, nf), st))) return rc;
        if ((rc = launch_select(dl, s_all + (size_t)h0 * L, k_keep, nullptr, nf, fb, idx, inv, st)))
            return rc;
        // C2 fused into the zero-row pass and the attention epilogue
        if ((rc = launch_gather_zero_rep(dl, k, v, idx, k_keep, at_ws(w.kc), at_ws(w.vc), inv,
                                         out_rep, st)))
            return rc;
        if ((rc = launch_attend_indexed_rep(dl, q, k, v, at_ws(w.kc), at_ws(w.vc), idx, k_keep,
                                            out_rep, st)))
            return rc;
        return launch_peer_barrier(peer->signals[1], world, rank, st);
    }
    // ---- NCCL form: in-place all-gathers of the score rows and the outputs
    const Nccl* n = nccl();
    if (!n) return invalid("tsa_sparse_attention_layer_sharded: libnccl.so.2 not available");
    if (!s_full || !out_full)
        return invalid("tsa_sparse_attention_layer_sharded: the NCCL form needs s_full and out_full");
    if (H % nh != 0) return invalid("tsa_sparse_attention_layer_sharded: uneven head shards");
    uint8_t* out_mine = static_cast<uint8_t*>(out_full) + (size_t)h0 * L * D * eb;
    const int dt = d->dtype == TSA_BF16 ? kNcclBfloat16 : kNcclFloat32;
    if (dense) {
        if ((rc = launch_write_int(k_keep, d->seq_len, st))) return rc;
        if ((rc = tsa_dense_attention(&dl, q, k, v, out_mine, st))) return rc;
    } else {
        float* s_mine = s_full + (size_t)h0 * L;
        if ((rc = score_stage(dl, q, k, single_replica(s_mine), ws, st))) return rc;
        if ((rc = nccl_check(n->all_gather(s_mine, s_full, (size_t)nh * L, kNcclFloat32, nccl_comm, st),
                             "ncclAllGather (scores)")))
            return rc;
        if ((rc = budget_stage(df, s_full, k_keep, ws, std::max(1, nf), st))) return rc;
        if ((rc = launch_select(dl, s_mine, k_keep, nullptr, nf, fb, idx, inv, st))) return rc;
        if (attend_sm100_supported(*d)) {
            if ((rc = launch_gather_zero(dl, q, k, v, idx, k_keep, nullptr, at_ws(w.kc), at_ws(w.vc),
                                         inv, out_mine, st)))
                return rc;
            if ((rc = launch_attend_indexed(dl, q, k, v, at_ws(w.kc), at_ws(w.vc), idx, k_keep,
                                            out_mine, st)))
                return rc;
        } else if ((rc = tsa_token_sparse_attention(&dl, q, k, v, idx, k_keep, out_mine, ws, st))) {
            return rc;
        }
    }
    return nccl_check(n->all_gather(out_mine, out_full, (size_t)nh * L * D, dt, nccl_comm, st),
                      "ncclAllGather (outputs)");
}
