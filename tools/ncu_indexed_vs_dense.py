"""Three attention launches for an ncu comparison at k_keep = L: the layer step
(indexed), dense, then indexed again on the same inputs."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2602_03216_b200 as tsa  # noqa: E402
from paper_2602_03216_b200 import workloads  # noqa: E402
from paper_2602_03216_b200.dist import ShardedSparseAttention  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
q, k, v = workloads.heavy_tailed_heads(32, 8, L, 128, seed=2602)
plan = tsa.SparsePlan(mode=tsa.SparseMode.kDynamic, sparse_layers=[0], tau=0.0)
lay = ShardedSparseAttention(32, 8, L, 128, torch.bfloat16, plan, device=q.device)
lay.step(q, k, v)
out = torch.empty_like(q)
lay.backend.dense(q, k, v, out)
lay.backend.attend_indexed(q, k, v, lay.backend.k_keep, out)
torch.cuda.synchronize()
