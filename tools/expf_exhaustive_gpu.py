"""Every float in [-104, 0] (and +0, -0, down to -inf-ish) through this build's
device expf vs the baseline build's, bitwise (argv[1]: baseline repo dir)."""
import ctypes as C
import sys
import torch
lo = 0x80000000  # -0.0
hi = 0xC2D00000  # -104.0
n = hi - lo + 1
libs = [C.CDLL(p + "/paper_2602_03216_b200/libtsa_b200.so") for p in (".", sys.argv[1])]
chunk = 1 << 28
bad = 0
for s in range(0, n, chunk):
    m = min(chunk, n - s)
    xi = torch.arange(lo + s, lo + s + m, dtype=torch.int64, device="cuda").to(torch.int32)
    x = xi.view(torch.float32)
    ys = []
    for L in libs:
        y = torch.empty_like(x)
        assert L.tsa_expf(C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), C.c_int64(m), None) == 0
        ys.append(y)
    torch.cuda.synchronize()
    bad += int((ys[0].view(torch.int32) != ys[1].view(torch.int32)).sum())
extra = torch.tensor([0.0, -1e-45, -1e-30, -2**-60, -2**-61, -105.0, -200.0, -float("inf")], device="cuda")
ys = []
for L in libs:
    y = torch.empty_like(extra)
    L.tsa_expf(C.c_void_p(extra.data_ptr()), C.c_void_p(y.data_ptr()), C.c_int64(extra.numel()), None)
    ys.append(y)
torch.cuda.synchronize()
print(f"expf exhaustive [-104, -0]: {n} inputs, {bad} mismatches; extras equal: {torch.equal(ys[0].view(torch.int32), ys[1].view(torch.int32))} {ys[0].tolist()}")
