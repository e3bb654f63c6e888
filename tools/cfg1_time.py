import torch, time, sys
sys.path.insert(0, '.')
import paper_2602_03216_b200 as tsa
from paper_2602_03216_b200 import workloads
q, k, v = workloads.uniform_heads(32, 8, 4096, 128, seed=11, dtype=torch.float32, device='cuda')
h = tsa.HeadTensors(q, k, v)
plan = tsa.SparsePlan(mode=tsa.SparseMode.kDynamic, sparse_layers=[0], tau=0.5)
out = torch.empty_like(q)
for _ in range(3): tsa.sparse_attention_layer(h, plan, out=out, stat=False)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20): tsa.sparse_attention_layer(h, plan, out=out, stat=False)
e.record(); torch.cuda.synchronize()
print('cfg1 layer ms', s.elapsed_time(e) / 20)
s.record()
for _ in range(20): tsa.sparse_attention_layer(h, tsa.SparsePlan(), out=out, stat=False)
e.record(); torch.cuda.synchronize()
print('cfg1 dense ms', s.elapsed_time(e) / 20)
