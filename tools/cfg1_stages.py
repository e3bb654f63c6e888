"""Per-stage times of cfg1 (4K fp32, 32/8 heads, tau = 0.5, REFERENCE-order scoring)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2602_03216_b200 as tsa  # noqa: E402
from paper_2602_03216_b200 import workloads  # noqa: E402
from paper_2602_03216_b200.dist import ShardedSparseAttention  # noqa: E402

L = 4096
q, k, v = workloads.uniform_heads(32, 8, L, 128, seed=2602, dtype=torch.float32)
plan = tsa.SparsePlan(mode=tsa.SparseMode.kDynamic, sparse_layers=[0], tau=0.5)
lay = ShardedSparseAttention(32, 8, L, 128, torch.float32, plan, device=q.device)
st = torch.cuda.current_stream()
for it in range(4):
    names, evs = [], []

    def mark(n):
        e = torch.cuda.Event(enable_timing=True)
        e.record(st)
        names.append(n)
        evs.append(e)
    lay.step(q, k, v, marks=mark)
    torch.cuda.synchronize()
    if it == 3:
        print({names[i]: round(evs[i - 1].elapsed_time(evs[i]), 3) for i in range(1, len(evs))},
              "k_keep", lay.k_keep)
