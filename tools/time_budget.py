"""Budget stage (headsum + the budget cluster kernel) at 128K / 32 heads on
realistic scores, exact total (REFERENCE scoring) vs the f64 tree (FAST):
CUDA events, after warm-up."""
import ctypes as C
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2602_03216_b200 as tsa  # noqa: E402
from paper_2602_03216_b200 import _lib, ops  # noqa: E402

H, L = 32, 131072
g = torch.Generator(device="cuda").manual_seed(0)
s = torch.exp(torch.randn((H, L), generator=g, device="cuda") * 2.5)
s = s / s.sum(1, keepdim=True) * 64
kk = torch.zeros(1, dtype=torch.int32, device="cuda")
for scoring, name in ((1, "exact"), (2, "fast")):
    d = ops._desc_for(H, 8, L, 128, _lib.TSA_BF16, mode=1, tau=0.01, scoring=scoring)
    ws = ops._workspace(d, torch.device("cuda"))
    st = ops._stream(torch.device("cuda"))
    f = lambda: _lib.check(_lib.load().tsa_budget(C.byref(d), ops._ptr(s), ops._ptr(kk), ops._ptr(ws), st))
    for _ in range(5):
        f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(50):
        f()
    b.record()
    torch.cuda.synchronize()
    print(name, "budget ms", round(a.elapsed_time(b) / 50, 4), "k_keep", int(kk.item()))
