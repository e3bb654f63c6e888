"""Attention-kernel-only timing (dense 128K and the sparse layer) for tuning."""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2602_03216_b200 as tsa  # noqa: E402
from paper_2602_03216_b200 import workloads  # noqa: E402
from paper_2602_03216_b200.dist import ShardedSparseAttention  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
q, k, v = workloads.heavy_tailed_heads(32, 8, L, 128, seed=2602)
dev = torch.device("cuda")
plan = tsa.SparsePlan(mode=tsa.SparseMode.kDynamic, sparse_layers=[0], tau=0.01)
lay = ShardedSparseAttention(32, 8, L, 128, torch.bfloat16, plan, device=dev)


def t(fn, n=4):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n


dense = t(lambda: lay.step(q, k, v, dense=True))
sparse = t(lambda: lay.step(q, k, v))
F = 2.0 * lay.k_keep * (lay.k_keep + 1) * 128 * 32
Fd = 2.0 * L * (L + 1) * 128 * 32
print(f"POLY={os.environ.get('TSA_EXP_POLY', 'default')} dense {dense:.2f} ms ({Fd/dense/1e9:.0f} TF/s) "
      f"sparse layer {sparse:.2f} ms  k={lay.k_keep} speedup {dense/sparse:.3f}", flush=True)
