"""One attention launch for ncu source-level capture (profiling only).
usage: ncu ... python tools/profile_attend.py [L] [dense|sparse]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2602_03216_b200 as tsa  # noqa: E402
from paper_2602_03216_b200 import workloads  # noqa: E402
from paper_2602_03216_b200.dist import ShardedSparseAttention  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
mode = sys.argv[2] if len(sys.argv) > 2 else "dense"
q, k, v = workloads.heavy_tailed_heads(32, 8, L, 128, seed=2602)
plan = tsa.SparsePlan(mode=tsa.SparseMode.kDynamic, sparse_layers=[0], tau=0.01)
lay = ShardedSparseAttention(32, 8, L, 128, torch.bfloat16, plan, device=torch.device("cuda"))
lay.step(q, k, v, dense=(mode == "dense"))
torch.cuda.synchronize()
