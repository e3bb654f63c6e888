"""The f32 attention on the tensor cores (attend_tf32.cu, 3xTF32) against a
float64 PyTorch reference of dense_causal_attention (attention.cpp:25-40), at
the reference's f32 gate max |d| <= 1e-5 (bench.cpp:27)."""
import math

import pytest
import torch

import paper_2602_03216_b200 as tsa
from tests import parity

pytestmark = pytest.mark.gpu


def ref_attention(q, k, v):
    """[n, d] float64 causal softmax(q k^T / sqrt(d)) v."""
    q, k, v = q.double(), k.double(), v.double()
    n = q.shape[0]
    s = (q @ k.t()) / math.sqrt(q.shape[1])
    s = s.masked_fill(torch.ones(n, n, dtype=torch.bool, device=q.device).triu(1), float("-inf"))
    return torch.softmax(s, dim=1) @ v


def uniform(shape, seed, lo=-1.0, hi=1.0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return torch.rand(shape, generator=g, device="cuda") * (hi - lo) + lo


@pytest.mark.parametrize("L", [1, 5, 127, 128, 129, 383, 1000, 2500])
def test_tf32_dense_head_vs_float64(cuda, L):
    q, k, v = (uniform((L, 128), s) for s in (1, 2, 3))
    out = tsa.dense_causal_attention(q, k, v)
    err = (out.double() - ref_attention(q, k, v)).abs().max().item()
    assert err <= parity.F32_GATE, err


@pytest.mark.parametrize("H,Hkv,L", [(4, 2, 700), (8, 1, 1500), (2, 2, 4096)])
def test_tf32_layer_dense_gqa(cuda, H, Hkv, L):
    q = uniform((H, L, 128), 4)
    k = uniform((Hkv, L, 128), 5)
    v = uniform((Hkv, L, 128), 6)
    out, st = tsa.sparse_attention_layer(tsa.HeadTensors(q, k, v), tsa.SparsePlan())
    for h in (0, H - 1):
        kv = h * Hkv // H
        err = (out[h].double() - ref_attention(q[h], k[kv], v[kv])).abs().max().item()
        assert err <= parity.F32_GATE, (h, err)


def test_tf32_sharp_logits_rescale(cuda):
    """Logits of +-60 that grow along the keys: the running max moves on every
    KV tile, so O is rescaled each time; exponentials far below the max vanish."""
    L = 1024
    u = torch.nn.functional.normalize(uniform((128,), 7), dim=0)
    ramp = torch.linspace(0.0, 1.0, L, device="cuda")[:, None]
    q = (60.0 * u).expand(L, 128).contiguous()
    k = (ramp * u * math.sqrt(128)) + 0.01 * uniform((L, 128), 8)
    v = uniform((L, 128), 9)
    out = tsa.dense_causal_attention(q, k, v)
    err = (out.double() - ref_attention(q, k, v)).abs().max().item()
    assert err <= parity.F32_GATE, err


def test_tf32_partial_tile_never_reads_the_next_head(cuda):
    """L = 300: head 0's last K/V tile is partial; the rows after it belong to
    head 1 and hold NaN.  The 3-D maps read zeros past the head, so head 0 is
    finite and within the gate (P = 0 times a NaN would poison it)."""
    L = 300
    q = uniform((2, L, 128), 10)
    k = uniform((2, L, 128), 11)
    v = uniform((2, L, 128), 12)
    k[1, :100] = float("nan")
    v[1, :100] = float("nan")
    out, _ = tsa.sparse_attention_layer(tsa.HeadTensors(q, k, v), tsa.SparsePlan())
    assert torch.isfinite(out[0]).all()
    err = (out[0].double() - ref_attention(q[0], k[0], v[0])).abs().max().item()
    assert err <= parity.F32_GATE, err


def test_tf32_sparse_layer_selected_rows(cuda, port):
    """The compressed path (gather -> tf32 attention -> scatter) vs the oracle on
    the same selection."""
    import numpy as np
    from oracle.oracle import RefRng, gqa_heads
    q, k, v = gqa_heads(RefRng(31), 4, 2, 1500, 128)
    h = tsa.HeadTensors(*(torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (q, k, v)))
    plan = tsa.SparsePlan(mode=tsa.SparseMode.kDynamic, sparse_layers=[0], tau=0.3)
    out, st = tsa.sparse_attention_layer(h, plan)
    idx = st.selection.indices.cpu().numpy().astype(np.int32)
    ref = port.token_sparse_attention(q, k, v, idx)
    assert np.abs(out.cpu().numpy() - ref).max() <= parity.F32_GATE
    assert parity.unselected_rows_zero(out.cpu().numpy(), idx, 1500)


@pytest.mark.parametrize("L", [100, 256, 385, 1000, 2047, 4096])
@pytest.mark.parametrize("pairs", ["0", "1"])
def test_tf32_single_and_pair_kernels(cuda, monkeypatch, L, pairs):
    """Both implementations (TSA_TF32_PAIRS: 2-CTA clusters sharing K / V halves,
    or one CTA per tile) at the gate, on odd and even tile counts (the last pair's
    upper tile absent) -- and they agree with each other to f32 rounding."""
    monkeypatch.setenv("TSA_TF32_PAIRS", pairs)
    q, k, v = (uniform((3, L, 128), s) for s in (21, 22, 23))
    out, _ = tsa.sparse_attention_layer(tsa.HeadTensors(q, k, v), tsa.SparsePlan())
    for h in range(3):
        err = (out[h].double() - ref_attention(q[h], k[h], v[h])).abs().max().item()
        assert err <= parity.F32_GATE, (h, err)
    monkeypatch.setenv("TSA_TF32_PAIRS", "1" if pairs == "0" else "0")
    other, _ = tsa.sparse_attention_layer(tsa.HeadTensors(q, k, v), tsa.SparsePlan())
    assert (out - other).abs().max().item() <= 2e-6
