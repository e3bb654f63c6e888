"""attend_indexed with the identity selection (k_keep = L) against the dense
kernel on the same inputs, alternating, CUDA events: isolates the per-CTA cost
of the indexed variant (Q load, scattered epilogue, in-place K/V maps)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2602_03216_b200 as tsa  # noqa: E402
from paper_2602_03216_b200 import workloads  # noqa: E402
from paper_2602_03216_b200.dist import ShardedSparseAttention  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
H, HKV = 32, 8
q, k, v = workloads.heavy_tailed_heads(H, HKV, L, 128, seed=2602)
dev = q.device
plan = tsa.SparsePlan(mode=tsa.SparseMode.kDynamic, sparse_layers=[0], tau=0.0)
lay = ShardedSparseAttention(H, HKV, L, 128, torch.bfloat16, plan, device=dev)
lay.step(q, k, v)  # selection = identity, k_keep = L
b = lay.backend
assert lay.k_keep == L
out = torch.empty_like(q)


def t(fn, n=10):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n


for rep in range(3):
    d = t(lambda: b.dense(q, k, v, out))
    i_ = t(lambda: b.attend_indexed(q, k, v, b.k_keep, out))
    print(f"L={L} dense {d:.3f} ms  indexed(identity, in place) {i_:.3f} ms  ratio {i_ / d:.3f}",
          flush=True)
