"""tsa_gather_zero on the bench's 128K selection, back to back (CUDA events):
compare with tools/probes/gather_probe (random selections, same shape)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2602_03216_b200 as tsa  # noqa: E402
from paper_2602_03216_b200 import workloads  # noqa: E402
from paper_2602_03216_b200.dist import ShardedSparseAttention  # noqa: E402

L = 131072
q, k, v = workloads.heavy_tailed_heads(32, 8, L, 128, seed=2602)
plan = tsa.SparsePlan(mode=tsa.SparseMode.kDynamic, sparse_layers=[0], tau=0.01)
lay = ShardedSparseAttention(32, 8, L, 128, torch.bfloat16, plan, device=q.device)
lay.step(q, k, v)
b = lay.backend
out = torch.empty_like(q)
for n_it in (1, 20):
    for _ in range(3):
        b.gather_kv_zero(k, v, b.k_keep, out)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n_it):
        b.gather_kv_zero(k, v, b.k_keep, out)
    e.record()
    torch.cuda.synchronize()
    print(f"gather_zero x{n_it}: {s.elapsed_time(e) / n_it:.3f} ms  k={lay.k_keep}")
# the same after the attention kernel (as in the step: select -> gather)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
tot = 0.0
for _ in range(5):
    b.attend_indexed(q, k, v, b.k_keep, out)
    s.record()
    b.gather_kv_zero(k, v, b.k_keep, out)
    e.record()
    torch.cuda.synchronize()
    tot += s.elapsed_time(e)
print(f"gather_zero after attention: {tot / 5:.3f} ms")
