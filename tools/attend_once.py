"""One cfg3 sparse layer (128K, exact scoring) for an ncu capture of the attention kernel."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2602_03216_b200 as tsa  # noqa: E402
from paper_2602_03216_b200 import workloads  # noqa: E402

q, k, v = workloads.heavy_tailed_heads(32, 8, 131072, 128, seed=2602, device="cuda")
plan = tsa.SparsePlan(mode=tsa.SparseMode.kDynamic, sparse_layers=[0], tau=0.01)
out, st = tsa.sparse_attention_layer(tsa.HeadTensors(q, k, v), plan)
torch.cuda.synchronize()
print("k_keep", st.k_keep)
