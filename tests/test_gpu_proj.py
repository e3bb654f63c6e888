"""The projections on the tensor cores (proj_gemm.cu): the plain tcgen05 GEMM,
project_qkv with rms_norm folded in (model.cpp:81-94, 128-158) and the W_O
projection + residual (model.cpp:196-201), each against a plain PyTorch fp32
reference of the same op.  bf16 inputs, f32 accumulation: the tolerance is the
output's bf16 rounding plus the f32 summation-order difference
(REL_L2 = 4e-3, max |err| <= 2^-7 |ref|max)."""
import math

import pytest
import torch

import paper_2602_03216_b200 as tsa

pytestmark = pytest.mark.gpu

REL_L2 = 4e-3
MAX_REL = 2.0 ** -7


def close(y, ref):
    y, ref = y.float(), ref.float()
    rel = ((y - ref).norm() / ref.norm().clamp_min(1e-30)).item()
    mx = (y - ref).abs().max().item() / ref.abs().max().clamp_min(1e-30).item()
    assert rel < REL_L2 and mx < MAX_REL, (rel, mx)


def rnd(*shape, seed=0, scale=1.0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return (torch.randn(shape, generator=g, device="cuda") * scale).to(torch.bfloat16)


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (300, 512, 256), (1024, 768, 4096),
                                   (4097, 256, 128)])
def test_gemm_bf16_vs_fp32(cuda, M, N, K):
    a, b = rnd(M, K, seed=1), rnd(N, K, seed=2)
    c = tsa.gemm_bf16(a, b)
    close(c, a.float() @ b.float().t())


def test_gemm_bf16_zero_inputs_and_shape_errors(cuda):
    c = tsa.gemm_bf16(torch.zeros((130, 64), dtype=torch.bfloat16, device="cuda"),
                      torch.zeros((256, 64), dtype=torch.bfloat16, device="cuda"))
    assert torch.count_nonzero(c) == 0
    with pytest.raises(tsa.InvalidArgument):  # N not a multiple of 256
        tsa.gemm_bf16(rnd(128, 64), rnd(200, 64))
    with pytest.raises(tsa.InvalidArgument):  # K not a multiple of 64
        tsa.gemm_bf16(rnd(128, 96), rnd(256, 96))


def test_gemm_bf16_many_tiles_persistent(cuda):
    """More tiles than SMs: every CTA walks several tiles through both TMEM accumulators."""
    a, b = rnd(128 * 40, 512, seed=3), rnd(256 * 9, 512, seed=4)
    close(tsa.gemm_bf16(a, b), a.float() @ b.float().t())


def test_prepare_weight_exact(cuda):
    w = torch.randn(96, 512, device="cuda")
    g = torch.rand(96, device="cuda") + 0.5
    wt = tsa.prepare_weight(w, g)
    ref = (w * g[:, None]).t().contiguous().to(torch.bfloat16)
    assert torch.equal(wt.view(torch.int16), ref.view(torch.int16))
    wb = w.to(torch.bfloat16)
    assert torch.equal(tsa.prepare_weight(wb).view(torch.int16), wb.t().contiguous().view(torch.int16))


def test_row_inv_rms(cuda):
    x = rnd(333, 4096, seed=5, scale=2.0)
    inv = tsa.row_inv_rms(x, 1e-5)
    ref = 1.0 / torch.sqrt(x.float().pow(2).mean(1) + 1e-5)
    assert torch.allclose(inv, ref, rtol=2e-6, atol=0)


def rope_ref(t, table):
    """apply_rope (model.cpp:107-126) on [rows, heads, d] f32 at positions 0..rows-1."""
    c, s = table[..., 0][:, None, :], table[..., 1][:, None, :]
    x0, x1 = t[..., 0::2], t[..., 1::2]
    out = torch.empty_like(t)
    out[..., 0::2] = x0 * c - x1 * s
    out[..., 1::2] = x0 * s + x1 * c
    return out


@pytest.mark.parametrize("L,H,Hkv,D", [(300, 4, 2, 512), (1024, 32, 8, 4096), (129, 2, 1, 128)])
def test_qkv_proj_vs_fp32(cuda, L, H, Hkv, D):
    """q/k/v = split_heads(rope(rms_norm(x, gain) W_qkv)) in one GEMM."""
    d = 128
    x = rnd(L, D, seed=6, scale=1.5)
    gain = torch.rand(D, device="cuda") + 0.5
    w = torch.randn(D, (H + 2 * Hkv) * d, device="cuda") / math.sqrt(D)
    table = tsa.rope_table(L, d, 500000.0, "cuda")
    eps = 1e-5
    heads = tsa.qkv_proj(x, tsa.prepare_weight(w, gain), tsa.row_inv_rms(x, eps), table, H, Hkv, d)
    xf = x.float()
    xn = xf / torch.sqrt(xf.pow(2).mean(1, keepdim=True) + eps) * gain
    p = (xn @ w).view(L, H + 2 * Hkv, d)
    p[:, :H + Hkv] = rope_ref(p[:, :H + Hkv], table)
    close(heads.q, p[:, :H].permute(1, 0, 2))
    close(heads.k, p[:, H:H + Hkv].permute(1, 0, 2))
    close(heads.v, p[:, H + Hkv:].permute(1, 0, 2))


def test_qkv_proj_matches_unfused_kernels(cuda):
    """Against the unfused stages (tsa.rms_norm -> cuBLAS -> tsa.split_heads_rope):
    the two differ only by where bf16 rounding happens."""
    L, H, Hkv, D, d = 512, 8, 2, 1024, 128
    x = rnd(L, D, seed=7)
    gain = torch.ones(D, device="cuda")
    w = (torch.randn(D, (H + 2 * Hkv) * d, device="cuda") / math.sqrt(D)).to(torch.bfloat16)
    table = tsa.rope_table(L, d, 10000.0, "cuda")
    fused = tsa.qkv_proj(x, tsa.prepare_weight(w, gain), tsa.row_inv_rms(x, 1e-5), table, H, Hkv, d)
    xn = tsa.rms_norm(x, gain, 1e-5)
    ref = tsa.split_heads_rope(xn @ w, table, H, Hkv, d)
    for a, b in ((fused.q, ref.q), (fused.k, ref.k), (fused.v, ref.v)):
        close(a, b)


def test_qkv_proj_without_norm(cuda):
    L, H, Hkv, D, d = 256, 2, 1, 256, 128
    x = rnd(L, D, seed=8)
    w = torch.randn(D, (H + 2 * Hkv) * d, device="cuda") / 16
    table = tsa.rope_table(L, d, 10000.0, "cuda")
    heads = tsa.qkv_proj(x, tsa.prepare_weight(w), None, table, H, Hkv, d)
    p = (x.float() @ w).view(L, H + 2 * Hkv, d)
    p[:, :H + Hkv] = rope_ref(p[:, :H + Hkv], table)
    close(heads.v, p[:, H + Hkv:].permute(1, 0, 2))
    close(heads.q, p[:, :H].permute(1, 0, 2))


@pytest.mark.parametrize("L,H,D", [(300, 4, 256), (1024, 32, 4096)])
def test_out_proj_residual_vs_fp32(cuda, L, H, D):
    """x += concat_h(o_h) W_o, A read from o [H, L, d] without a concat buffer."""
    d = 128
    o = rnd(H, L, d, seed=9)
    wo = torch.randn(H * d, D, device="cuda") / math.sqrt(H * d)
    x = rnd(L, D, seed=10)
    ref = x.float() + o.permute(1, 0, 2).reshape(L, H * d).float() @ wo
    tsa.out_proj_residual(o, tsa.prepare_weight(wo), x)
    close(x, ref)


def test_out_proj_matches_concat_addmm(cuda):
    L, H, D, d = 512, 8, 1024, 128
    o = rnd(H, L, d, seed=11)
    wo = (torch.randn(H * d, D, device="cuda") / 32).to(torch.bfloat16)
    x = rnd(L, D, seed=12)
    x2 = x.clone()
    tsa.out_proj_residual(o, tsa.prepare_weight(wo), x)
    x2.addmm_(tsa.heads_concat(o), wo)
    close(x, x2)


def test_projections_at_cfg4_size_sampled_rows(cuda):
    """cfg4's per-layer shapes (L = 65536, d_model 4096, 32 / 8 heads): the fused
    QKV projection and the W_o projection + residual, sampled rows against fp32
    (the kernels run every tile; the check reads 512 rows spread over L, so
    every M tile position class and all N tiles are covered)."""
    L, D, H, Hkv, d = 65536, 4096, 32, 8, 128
    x = rnd(L, D, seed=20)
    gain = torch.rand(D, device="cuda") + 0.5
    w = (torch.randn(D, (H + 2 * Hkv) * d, device="cuda") / math.sqrt(D)).to(torch.bfloat16)
    table = tsa.rope_table(L, d, 500000.0, "cuda")
    heads = tsa.qkv_proj(x, tsa.prepare_weight(w, gain), tsa.row_inv_rms(x, 1e-5), table, H,
                         Hkv, d)
    rows = torch.linspace(0, L - 1, 512, device="cuda").long()
    xf = x[rows].float()
    xn = xf / torch.sqrt(xf.pow(2).mean(1, keepdim=True) + 1e-5) * gain
    p = (xn @ w.float()).view(-1, H + 2 * Hkv, d)
    p[:, :H + Hkv] = rope_ref(p[:, :H + Hkv], table[rows])
    close(heads.q[:, rows], p[:, :H].permute(1, 0, 2))
    close(heads.k[:, rows], p[:, H:H + Hkv].permute(1, 0, 2))
    close(heads.v[:, rows], p[:, H + Hkv:].permute(1, 0, 2))
    wo = (torch.randn(H * d, D, device="cuda") / math.sqrt(H * d)).to(torch.bfloat16)
    o = heads.q
    x0 = x[rows].float()
    tsa.out_proj_residual(o, tsa.prepare_weight(wo), x)
    ref = x0 + o[:, rows].permute(1, 0, 2).reshape(-1, H * d).float() @ wo.float()
    close(x[rows], ref)


def test_projection_argument_errors(cuda):
    """Misaligned buffers and wrong dtypes fail loudly (no fault, no silent garbage)."""
    a = rnd(129, 64)
    b = rnd(256, 64)
    c = torch.empty(129 * 256 + 1, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(tsa.InvalidArgument):  # c offset by one element: not 16-B aligned
        tsa.gemm_bf16(a, b, out=c[1:].view(129, 256))
    x = rnd(64, 256)
    table = tsa.rope_table(64, 128, 10000.0, "cuda")
    with pytest.raises(tsa.InvalidArgument):  # f32 weights
        tsa.qkv_proj(x, torch.zeros((512, 256), device="cuda"), None, table, 2, 1, 128)
    with pytest.raises(tsa.InvalidArgument):
        tsa.out_proj_residual(rnd(2, 64, 128), torch.zeros((256, 256), device="cuda"), x)
