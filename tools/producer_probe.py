"""Times the cfg4 producer stages at L = 64K (diagnostics)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2602_03216_b200 as tsa  # noqa: E402
from paper_2602_03216_b200.stack import structured_hidden  # noqa: E402

L, D, H, Hkv, d = 65536, 4096, 32, 8, 128
x = structured_hidden(L, D, seed=1)
g = torch.ones(D, device="cuda")
w = torch.randn((D, (H + 2 * Hkv) * d), device="cuda").to(torch.bfloat16) * 0.02
xn = torch.empty_like(x)
qkv = torch.empty((L, (H + 2 * Hkv) * d), dtype=torch.bfloat16, device="cuda")
table = tsa.rope_table(L, d, 500000.0, "cuda")
ht = tsa.split_heads_rope(qkv, table, H, Hkv, d)
cat = torch.empty((L, H * d), dtype=torch.bfloat16, device="cuda")
wo = torch.randn((H * d, D), device="cuda").to(torch.bfloat16) * 0.02


def t(fn, n=5):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n


print("rms_norm", round(t(lambda: tsa.rms_norm(x, g, 1e-5, out=xn)), 3), "ms")
print("qkv gemm", round(t(lambda: torch.matmul(xn, w, out=qkv)), 3), "ms")
print("split_rope", round(t(lambda: tsa.split_heads_rope(qkv, table, H, Hkv, d, out=ht)), 3), "ms")
print("concat", round(t(lambda: tsa.heads_concat(ht.q, out=cat)), 3), "ms")
print("wo gemm+res", round(t(lambda: x.addmm_(cat, wo)), 3), "ms")
