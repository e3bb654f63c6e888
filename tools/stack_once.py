"""cfg4's 32-layer stack (64K, Llama-3-8B heads, d_model 4096), one warm forward then
one forward for an ncu launch list: python tools/stack_once.py [--layers 32]"""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2602_03216_b200 as tsa  # noqa: E402
from paper_2602_03216_b200.stack import PrefillAttentionStack, structured_hidden  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=32)
ap.add_argument("--L", type=int, default=65536)
a = ap.parse_args()
plan = tsa.SparsePlan(mode=tsa.SparseMode.kDynamic, sparse_layers=list(range(a.layers)), tau=0.01)
st = PrefillAttentionStack(a.layers, 32, 8, 128, 4096, a.L, plan, seed=4, device="cuda")
x0 = structured_hidden(a.L, 4096, seed=5)
x = x0.clone()
st.forward(x)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
x.copy_(x0)
ev[0].record()
st.forward(x)
ev[1].record()
torch.cuda.synchronize()
print("forward ms", round(ev[0].elapsed_time(ev[1]), 1), "k_keep", st.k_keep.cpu().tolist())
x.copy_(x0)
st.forward_graphed(x)  # eager + capture
torch.cuda.synchronize()
x.copy_(x0)
ev[0].record()
st.forward_graphed(x)
ev[1].record()
torch.cuda.synchronize()
print("graphed forward ms", round(ev[0].elapsed_time(ev[1]), 1))
