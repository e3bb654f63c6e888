"""A/B helper for the exact scorer: times scoring (default mode) at 128K with CUDA
events and checks the scores bitwise against a reference file written by the
first build run (python tools/score_variant.py REF_PATH)."""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path.cwd()))
import paper_2602_03216_b200 as tsa  # noqa: E402
from paper_2602_03216_b200 import workloads  # noqa: E402

ref = sys.argv[1]
q, k, v = workloads.heavy_tailed_heads(32, 8, 131072, 128, seed=2602)
h = tsa.HeadTensors(q, k, v)
s = tsa.score_tokens(h, 64, 7).s.clone()
torch.cuda.synchronize()
ts = []
for _ in range(15):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    tsa.score_tokens(h, 64, 7)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
if not os.path.exists(ref):
    torch.save(s.cpu(), ref)
    same = "ref written"
else:
    r = torch.load(ref)
    same = bool(torch.equal(r.view(torch.int32), s.cpu().view(torch.int32)))
ts.sort()
print(f"{Path.cwd().name}: score min {ts[0]:.3f} med {ts[len(ts)//2]:.3f} ms bit-identical={same}")
