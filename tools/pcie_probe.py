"""PCIe copy rates on the box: pinned H2D of cfg3's inputs (1.5 GiB), D2H of its
output (1 GiB), alone and concurrently (two streams), CUDA events."""
import torch

n_in, n_out = 1610612736, 1073741824
h_in = torch.empty(n_in, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n_out, dtype=torch.uint8).pin_memory()
d_in = torch.empty(n_in, dtype=torch.uint8, device="cuda")
d_out = torch.empty(n_out, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b)


def both():
    e = torch.cuda.Event()
    e.record()
    s1.wait_event(e)
    s2.wait_event(e)
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


h2d = t(lambda: d_in.copy_(h_in, non_blocking=True))
d2h = t(lambda: h_out.copy_(d_out, non_blocking=True))
bi = t(both)
print(f"H2D {n_in / h2d / 1e6:.1f} GB/s ({h2d:.2f} ms), D2H {n_out / d2h / 1e6:.1f} GB/s "
      f"({d2h:.2f} ms), both at once {bi:.2f} ms")
