"""cfg4 producer / consumer timing: the hand-written tcgen05 projections
(proj_gemm.cu) against cuBLAS (torch.matmul) and the unfused stage chains, at
cfg4's per-layer shapes (L = 65536, d_model 4096, 32 / 8 heads, d = 128).

  python tools/proj_bench.py [--L 65536] [--iters 20]

CUDA events on the current stream, after warm-up; inputs (0.5 GB + weights)
are larger than what one iteration's tiles keep in L2."""
import argparse
import json
import math
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2602_03216_b200 as tsa  # noqa: E402


def timed(fn, iters):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--L", type=int, default=65536)
    ap.add_argument("--D", type=int, default=4096)
    ap.add_argument("--H", type=int, default=32)
    ap.add_argument("--Hkv", type=int, default=8)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--once", action="store_true",
                    help="one call of each fused projection, untimed (for ncu)")
    args = ap.parse_args()
    L, D, H, Hkv, d = args.L, args.D, args.H, args.Hkv, 128
    Nqkv = (H + 2 * Hkv) * d
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn((L, D), generator=g, device="cuda").to(torch.bfloat16)
    w = (torch.randn((D, Nqkv), generator=g, device="cuda") / math.sqrt(D)).to(torch.bfloat16)
    wo = (torch.randn((H * d, D), generator=g, device="cuda") / math.sqrt(H * d)).to(torch.bfloat16)
    gain = torch.ones(D, device="cuda")
    w_t, wo_t = tsa.prepare_weight(w, gain), tsa.prepare_weight(wo)
    table = tsa.rope_table(L, d, 500000.0, "cuda")
    inv = torch.empty(L, dtype=torch.float32, device="cuda")
    heads = tsa.HeadTensors(torch.empty((H, L, d), dtype=torch.bfloat16, device="cuda"),
                            torch.empty((Hkv, L, d), dtype=torch.bfloat16, device="cuda"),
                            torch.empty((Hkv, L, d), dtype=torch.bfloat16, device="cuda"))
    xn = torch.empty_like(x)
    qkv = torch.empty((L, Nqkv), dtype=torch.bfloat16, device="cuda")
    cat = torch.empty((L, H * d), dtype=torch.bfloat16, device="cuda")
    o = torch.randn((H, L, d), generator=g, device="cuda").to(torch.bfloat16)
    c_qkv = torch.empty((L, Nqkv), dtype=torch.bfloat16, device="cuda")
    c_o = torch.empty((L, D), dtype=torch.bfloat16, device="cuda")
    xr = x.clone()
    if args.once:
        tsa.row_inv_rms(x, 1e-5, out=inv)
        tsa.qkv_proj(x, w_t, inv, table, H, Hkv, d, out=heads)
        tsa.out_proj_residual(o, wo_t, xr)
        torch.cuda.synchronize()
        return
    it = args.iters
    f_qkv = 2.0 * L * D * Nqkv
    f_o = 2.0 * L * H * d * D
    r = {}
    r["gemm_qkv_tsa_ms"] = timed(lambda: tsa.gemm_bf16(x, w_t, out=c_qkv), it)
    r["gemm_qkv_cublas_ms"] = timed(lambda: torch.matmul(x, w, out=qkv), it)
    r["gemm_o_tsa_ms"] = timed(lambda: tsa.gemm_bf16(cat, wo_t, out=c_o), it)
    r["gemm_o_cublas_ms"] = timed(lambda: torch.matmul(cat, wo, out=c_o), it)
    r["inv_rms_ms"] = timed(lambda: tsa.row_inv_rms(x, 1e-5, out=inv), it)
    r["qkv_fused_ms"] = timed(lambda: tsa.qkv_proj(x, w_t, inv, table, H, Hkv, d, out=heads), it)

    def unfused_producer():
        tsa.rms_norm(x, gain, 1e-5, out=xn)
        torch.matmul(xn, w, out=qkv)
        tsa.split_heads_rope(qkv, table, H, Hkv, d, out=heads)

    def fused_producer():
        tsa.row_inv_rms(x, 1e-5, out=inv)
        tsa.qkv_proj(x, w_t, inv, table, H, Hkv, d, out=heads)

    r["producer_unfused_ms"] = timed(unfused_producer, it)
    r["producer_fused_ms"] = timed(fused_producer, it)
    r["out_fused_ms"] = timed(lambda: tsa.out_proj_residual(o, wo_t, xr), it)

    def unfused_consumer():
        tsa.heads_concat(o, out=cat)
        xr.addmm_(cat, wo)

    r["consumer_unfused_ms"] = timed(unfused_consumer, it)
    for k in ("gemm_qkv_tsa", "gemm_qkv_cublas", "qkv_fused"):
        r[k + "_TFLOP/s"] = round(f_qkv / r[k + "_ms"] / 1e9, 1)
    for k in ("gemm_o_tsa", "gemm_o_cublas", "out_fused"):
        r[k + "_TFLOP/s"] = round(f_o / r[k + "_ms"] / 1e9, 1)
    r = {k: (round(v, 4) if isinstance(v, float) else v) for k, v in r.items()}
    r["shape"] = dict(L=L, D=D, H=H, Hkv=Hkv, d=d)
    print(json.dumps(r))


if __name__ == "__main__":
    main()
