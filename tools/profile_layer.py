"""One sparse-layer step (128K Llama-3-8B, tau 0.01, default scoring) for ncu:
  ncu --set full --clock-control none -o out python tools/profile_layer.py
Runs the stage-by-stage step once (eager, so every kernel is its own launch)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2602_03216_b200 as tsa  # noqa: E402
from paper_2602_03216_b200 import workloads  # noqa: E402
from paper_2602_03216_b200.dist import ShardedSparseAttention  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
scoring = int(sys.argv[2]) if len(sys.argv) > 2 else 0
q, k, v = workloads.heavy_tailed_heads(32, 8, L, 128, seed=2602)
plan = tsa.SparsePlan(mode=tsa.SparseMode.kDynamic, sparse_layers=[0], tau=0.01)
lay = ShardedSparseAttention(32, 8, L, 128, torch.bfloat16, plan, device=q.device, scoring=scoring)
lay.step(q, k, v, marks=lambda name: None)
torch.cuda.synchronize()
print("k_keep", lay.k_keep)
