"""One 128K sparse layer under ncu (profiling only; numbers from this run are
never bench values).  usage: ncu ... python tools/profile_layer.py [L]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2602_03216_b200 as tsa  # noqa: E402
from paper_2602_03216_b200 import workloads  # noqa: E402
from paper_2602_03216_b200.dist import ShardedSparseAttention  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
H = int(sys.argv[2]) if len(sys.argv) > 2 else 32
HKV = int(sys.argv[3]) if len(sys.argv) > 3 else 8
q, k, v = workloads.heavy_tailed_heads(H, HKV, L, 128, seed=2602)
plan = tsa.SparsePlan(mode=tsa.SparseMode.kDynamic, sparse_layers=[0], tau=0.01)
lay = ShardedSparseAttention(H, HKV, L, 128, torch.bfloat16, plan, device=torch.device("cuda"))
for _ in range(2):
    lay.step(q, k, v)
torch.cuda.synchronize()
print("k_keep", lay.k_keep)
