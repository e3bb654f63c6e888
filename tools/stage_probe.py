"""Times each stage of the sparse layer at a given L (diagnostics)."""
import faulthandler
import sys
import time

import torch

sys.path.insert(0, ".")
faulthandler.dump_traceback_later(int(sys.argv[2]) if len(sys.argv) > 2 else 120, exit=True)
import paper_2602_03216_b200 as tsa  # noqa: E402
from paper_2602_03216_b200 import workloads  # noqa: E402
from paper_2602_03216_b200.dist import ShardedSparseAttention  # noqa: E402

L = int(sys.argv[1])
gen = sys.argv[3] if len(sys.argv) > 3 else "heavy"
tau = float(sys.argv[4]) if len(sys.argv) > 4 else 0.01
if gen == "uniform":
    q, k, v = workloads.uniform_heads(32, 8, L, 128, seed=2602)
else:
    q, k, v = workloads.heavy_tailed_heads(32, 8, L, 128, seed=2602)
dev = torch.device("cuda")
for scoring in (2, 1):
    plan = tsa.SparsePlan(mode=tsa.SparseMode.kDynamic, sparse_layers=[0], tau=tau)
    lay = ShardedSparseAttention(32, 8, L, 128, torch.bfloat16, plan, device=dev, scoring=scoring)
    for it in range(3):
        names, evs = [], []

        def mark(n):
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            names.append(n)
            evs.append(e)
        t0 = time.time()
        lay.step(q, k, v, marks=mark)
        torch.cuda.synchronize()
        st = {names[i]: round(evs[i - 1].elapsed_time(evs[i]), 3) for i in range(1, len(evs))}
        print(f"L={L} scoring={scoring} it={it} k_keep={lay.k_keep} wall={time.time()-t0:.3f}s {st}",
              flush=True)
    del lay
lay = ShardedSparseAttention(32, 8, L, 128, torch.bfloat16, tsa.SparsePlan(), device=dev)
for it in range(2):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    lay.step(q, k, v, dense=True)
    e.record()
    torch.cuda.synchronize()
    print(f"L={L} dense {s.elapsed_time(e):.3f} ms", flush=True)
