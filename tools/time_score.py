"""Times the scoring modes at a given size with CUDA events (per-kernel split
from the library's stage calls), e.g. python tools/time_score.py --seq-len 131072"""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2602_03216_b200 as tsa  # noqa: E402
from paper_2602_03216_b200 import workloads  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--seq-len", type=int, default=131072)
p.add_argument("--heads", type=int, default=32)
p.add_argument("--kv-heads", type=int, default=8)
p.add_argument("--reps", type=int, default=5)
p.add_argument("--modes", default="2,1")
a = p.parse_args()
q, k, v = workloads.heavy_tailed_heads(a.heads, a.kv_heads, a.seq_len, 128, seed=2602)
h = tsa.HeadTensors(q, k, v)
res = {}
for mode in [int(m) for m in a.modes.split(",")]:
    s = tsa.score_tokens(h, 64, 7, scoring=mode).s
    torch.cuda.synchronize()
    ts = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        tsa.score_tokens(h, 64, 7, scoring=mode)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    res[mode] = (min(ts), s)
    print(f"scoring={mode}: min {min(ts):.3f} ms, all {[round(t, 3) for t in ts]}")
if 1 in res and 2 in res:
    a_, b_ = res[1][1], res[2][1]
    rel = ((a_ - b_).abs() / a_.abs().clamp_min(1e-30))
    big = a_ > 1e-6 * a_.max()
    print(f"FAST vs EXACT: max rel {rel[big].max().item():.3e}, "
          f"bit-identical {(a_.view(torch.int32) == b_.view(torch.int32)).float().mean().item():.4f}")
