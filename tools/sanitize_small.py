"""Small end-to-end runs of every production path, for compute-sanitizer:
FAST bf16 layer (fused gather/attend), tau = 0 in-place, fixed mode, f32
reference-order layer, host-tensor pipeline, dense, producer kernels."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2602_03216_b200 as tsa  # noqa: E402
from paper_2602_03216_b200 import workloads  # noqa: E402

for L in (1000, 1537):
    q, k, v = workloads.heavy_tailed_heads(8, 2, L, 128, seed=3)
    h = tsa.HeadTensors(q, k, v)
    for plan in (tsa.SparsePlan(mode=tsa.SparseMode.kDynamic, sparse_layers=[0], tau=0.02),
                 tsa.SparsePlan(mode=tsa.SparseMode.kDynamic, sparse_layers=[0], tau=0.0),
                 tsa.SparsePlan(mode=tsa.SparseMode.kFixed, sparse_layers=[0], s_fixed=0.5),
                 tsa.SparsePlan()):
        out, st = tsa.sparse_attention_layer(h, plan)
        hq, hk, hv = (t.cpu().pin_memory() for t in (q, k, v))
        hout = torch.empty(q.shape, dtype=q.dtype).pin_memory()
        tsa.sparse_attention_layer_host(hq, hk, hv, hout, plan, n_groups=2)
    hf = tsa.HeadTensors(q.float(), k.float(), v.float())
    tsa.sparse_attention_layer(hf, tsa.SparsePlan(mode=tsa.SparseMode.kDynamic, sparse_layers=[0],
                                                  tau=0.3))
torch.cuda.synchronize()
print("sanitize_small done")
