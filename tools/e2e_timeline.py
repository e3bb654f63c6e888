"""Timeline of one host-tensor layer call (tsa_sparse_attention_layer_host) at
cfg3: CUPTI (torch.profiler) records every copy and kernel on every stream;
prints when the copies finish, when each stage runs, and the idle gaps of the
compute stream."""
import sys
from pathlib import Path

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2602_03216_b200 as tsa  # noqa: E402
from paper_2602_03216_b200 import workloads  # noqa: E402

H, Hkv, L, D = 32, 8, 131072, 128
q, k, v = workloads.heavy_tailed_heads(H, Hkv, L, D, seed=2602, device="cuda")
qh, kh, vh = (t.cpu().pin_memory() for t in (q, k, v))
oh = torch.empty_like(qh).pin_memory()
del q, k, v
plan = tsa.SparsePlan(mode=tsa.SparseMode.kDynamic, sparse_layers=[0], tau=0.01)
for _ in range(2):
    tsa.sparse_attention_layer_host(qh, kh, vh, oh, plan)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    tsa.sparse_attention_layer_host(qh, kh, vh, oh, plan)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
t0 = min(e.time_range.start for e in ev)
rows = sorted(((e.time_range.start - t0) / 1e3, (e.time_range.end - t0) / 1e3, e.name) for e in ev)
end = max(r[1] for r in rows)
print(f"events {len(rows)}, span {end:.2f} ms")
h2d = [r for r in rows if "HtoD" in r[2]]
d2h = [r for r in rows if "DtoH" in r[2]]
ker = [r for r in rows if "Memcpy" not in r[2] and "Memset" not in r[2]]
print(f"H2D {h2d[0][0]:.2f} .. {h2d[-1][1]:.2f} ms ({len(h2d)} copies); D2H {d2h[0][0]:.2f} .. {d2h[-1][1]:.2f}")
first_attend = next(r for r in ker if "attend" in r[2])
print(f"first attend at {first_attend[0]:.2f} ms; last kernel ends {ker[-1][1]:.2f} ms")
busy, last = 0.0, 0.0
gaps = []
for s, e, n in ker:
    if s > last + 0.05:
        gaps.append((last, s))
    busy += max(0.0, e - max(s, last))
    last = max(last, e)
print(f"kernel busy {busy:.2f} ms; gaps > 50 us: " + ", ".join(f"{a:.2f}-{b:.2f}" for a, b in gaps[:20]))
for s, e, n in ker:
    if "attend" in n or "budget" in n or "select" in n or "gather" in n:
        print(f"  {s:8.2f} {e:8.2f} {n[:60]}")

# back to back, as the bench's e2e times it: the gap between one call's last
# copy back and the next call's first copy in
import time  # noqa: E402
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof2:
    t_host = []
    for _ in range(3):
        a = time.perf_counter()
        tsa.sparse_attention_layer_host(qh, kh, vh, oh, plan)
        t_host.append((time.perf_counter() - a) * 1e3)
    torch.cuda.synchronize()
ev = [e for e in prof2.events() if e.device_type.name == "CUDA"]
t0 = min(e.time_range.start for e in ev)
cp = sorted(((e.time_range.start - t0) / 1e3, (e.time_range.end - t0) / 1e3, e.name) for e in ev
            if "Memcpy" in e.name)
print("host ms per call:", [round(x, 2) for x in t_host])
print(f"3 calls span {max(r[1] for r in cp):.2f} ms")
h2d = [r for r in cp if "HtoD" in r[2]]
d2h = [r for r in cp if "DtoH" in r[2]]
# calls: a new call starts where an H2D begins more than 1 ms after the previous H2D ended
starts = [h2d[0][0]] + [b[0] for a, b in zip(h2d, h2d[1:]) if b[0] - a[1] > 1.0]
print("call starts (first H2D):", [round(x, 2) for x in starts])
print("D2H ends:", [round(e_, 2) for s_, e_, n in d2h if e_ > 0][-1])
