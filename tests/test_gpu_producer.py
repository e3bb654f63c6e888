"""Parity of the attention-branch producer/consumer kernels (rms_norm,
RoPE + head split, head concat; model.cpp:81-158, 196-200) against the CPU
oracle (pinned bit-exact to the reference's model.cpp), and of the cfg4 layer
stack against a composition of those stages.  Runs on the B200 box: -m gpu."""
import numpy as np
import pytest
import torch

import paper_2602_03216_b200 as tsa
from oracle.oracle import RefRng
from tests import parity

pytestmark = pytest.mark.gpu


def dev(a, dtype=torch.float32):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dtype)


def host(t):
    return t.detach().float().cpu().numpy()


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


@pytest.mark.parametrize("rows,cols,eps", [(300, 96, 1e-5), (129, 4096, 1e-5), (7, 16, 0.0),
                                           (1, 1, 1e-5)])
def test_rms_norm_f32_bit_exact(cuda, port, rows, cols, eps):
    """model.cpp:81-94: sequential f32 sum of squares, (x * inv) * gain."""
    rng = RefRng(rows + cols)
    x = rng.random_matrix(rows, cols, 3.0)
    g = rng.random_matrix(1, cols, 2.0).reshape(-1)
    y = host(tsa.rms_norm(dev(x), dev(g), eps))
    assert np.array_equal(bits(y), bits(port.rms_norm(x, g, eps)))


def test_rms_norm_bf16_is_the_rounded_f32_result(cuda, port):
    rng = RefRng(5)
    xb = dev(rng.random_matrix(64, 512, 2.0), torch.bfloat16)
    g = rng.random_matrix(1, 512, 1.0).reshape(-1)
    y = tsa.rms_norm(xb, dev(g), 1e-5)
    ref = torch.from_numpy(port.rms_norm(host(xb), g, 1e-5)).to(torch.bfloat16)
    assert torch.equal(y.cpu().view(torch.int16), ref.view(torch.int16))


def test_rms_norm_zero_rows_and_gain_mismatch(cuda):
    y = host(tsa.rms_norm(torch.zeros((2, 4), device="cuda"), torch.ones(4, device="cuda"), 1e-5))
    assert np.all(y == 0.0)
    with pytest.raises(tsa.InvalidArgument):
        tsa.rms_norm(torch.zeros((2, 4), device="cuda"), torch.ones(3, device="cuda"), 1e-5)


@pytest.mark.parametrize("L,H,Hkv,d,theta", [(300, 4, 2, 64, 10000.0), (2048, 8, 2, 128, 500000.0),
                                             (1, 2, 1, 16, 10000.0)])
def test_split_heads_rope_vs_oracle(cuda, port, L, H, Hkv, d, theta):
    """split_heads + apply_rope (model.cpp:128-158): v copied exactly, q and k
    rotated with the reference's f32 arithmetic; cos/sin are the double libm
    results rounded to f32, equal to the host's except at rare 1-ulp ties."""
    rng = RefRng(L + d)
    W = (H + 2 * Hkv) * d
    qkv = rng.random_matrix(L, W, 2.0)
    table = tsa.rope_table(L, d, theta, "cuda")
    ht = tsa.split_heads_rope(dev(qkv), table, H, Hkv, d)
    parts = [(host(ht.q), 0, H, True), (host(ht.k), H, Hkv, True), (host(ht.v), H + Hkv, Hkv, False)]
    for out, s0, n, rot in parts:
        for h in range(n):
            src = qkv[:, (s0 + h) * d:(s0 + h + 1) * d]
            ref = port.apply_rope(src, theta) if rot else src
            o = out[h]
            same = np.mean(bits(o) == bits(ref))
            assert same >= 0.999, same
            np.testing.assert_allclose(o, ref, rtol=2 * 2**-23, atol=2 * 2**-23 * np.abs(src).max())


def test_rope_position_zero_identity_and_relative_dot(cuda):
    """test_model.cpp:110-148 on the GPU rotation."""
    d, L = 64, 512
    table = tsa.rope_table(L, d, 10000.0, "cuda")
    rng = RefRng(3)
    qrow, krow = rng.random_matrix(1, d, 1.0), rng.random_matrix(1, d, 1.0)
    qkv = np.concatenate([np.tile(qrow, (L, 1)), np.tile(krow, (L, 1)), np.zeros((L, d), np.float32)],
                         axis=1)
    ht = tsa.split_heads_rope(dev(qkv), table, 1, 1, d)
    q, k = host(ht.q)[0], host(ht.k)[0]
    assert np.array_equal(bits(q[0]), bits(qrow[0]))
    d1, d2 = float(q[300] @ k[200]), float(q[150] @ k[50])
    assert abs(d1 - d2) < 1e-4 * max(1.0, abs(d1))


def test_heads_concat_exact(cuda):
    x = torch.randn((4, 100, 128), device="cuda").to(torch.bfloat16)
    cat = tsa.heads_concat(x)
    assert torch.equal(cat, x.permute(1, 0, 2).reshape(100, 4 * 128))
    xf = torch.randn((3, 17, 8), device="cuda")
    assert torch.equal(tsa.heads_concat(xf), xf.permute(1, 0, 2).reshape(17, 24))


def _stack(L, n_layers=2, tau=0.01, seed=0):
    from paper_2602_03216_b200.stack import PrefillAttentionStack
    plan = tsa.SparsePlan(mode=tsa.SparseMode.kDynamic, sparse_layers=list(range(n_layers)),
                          tau=tau)
    return PrefillAttentionStack(n_layers, 8, 2, 128, 512, L, plan, seed=seed, device="cuda")


def test_stack_layer_is_the_composition_of_the_stages(cuda):
    """One stack layer == row_inv_rms -> qkv_proj (rms scale, GEMM, RoPE, split)
    -> sparse layer -> out_proj_residual, step by step through the public
    operators (bitwise); and within bf16 tolerance of the unfused chain
    rms_norm -> cuBLAS -> split/RoPE -> sparse layer -> concat -> x + cat W_o
    (the selection may differ by near-ties, so the unfused chain runs on the
    fused chain's selection: the dense-layer output is compared)."""
    from paper_2602_03216_b200.stack import structured_hidden
    L = 1024
    st = _stack(L)
    x = structured_hidden(L, 512, seed=1)
    x0 = x.clone()
    st.layer(0, x)
    w = st.layers[0]
    inv = tsa.row_inv_rms(x0, 1e-5)
    ht = tsa.qkv_proj(x0, w.wqkv_t, inv, st.table, 8, 2, 128)
    plan = tsa.SparsePlan(mode=tsa.SparseMode.kDynamic, sparse_layers=[0], tau=0.01)
    o, stat = tsa.sparse_attention_layer(ht, plan)
    ref = x0.clone()
    tsa.out_proj_residual(o, w.wo_t, ref)
    assert int(st.k_keep[0].item()) == stat.k_keep < L
    assert torch.equal(x.view(torch.int16), ref.view(torch.int16))
    # unfused: the same dense layer through the separate stages and cuBLAS
    xd = x0.clone()
    st.layer(0, xd, dense=True)
    hu = tsa.split_heads_rope(tsa.rms_norm(x0, w.attn_norm, 1e-5) @ w.wqkv, st.table, 8, 2, 128)
    for a, b in ((ht.q, hu.q), (ht.k, hu.k), (ht.v, hu.v)):
        rel = ((a.float() - b.float()).norm() / b.float().norm()).item()
        assert rel < 4e-3, rel
    dense = tsa.SparsePlan(mode=tsa.SparseMode.kDynamic, sparse_layers=[0], tau=0.0)  # keep all
    of, _ = tsa.sparse_attention_layer(ht, dense)
    ou, _ = tsa.sparse_attention_layer(hu, dense)
    rel_o = ((of.float() - ou.float()).norm() / ou.float().norm()).item()
    assert rel_o < 1e-2, rel_o
    # the consumer on the same attention output (the softmax amplifies the
    # producer's rounding differences, so xd itself is not compared)
    xu = x0.clone()
    xu.addmm_(tsa.heads_concat(ou), w.wo)
    xf = x0.clone()
    tsa.out_proj_residual(ou, w.wo_t, xf)
    rel_x = ((xf.float() - xu.float()).norm() / xu.float().norm()).item()
    assert rel_x < 4e-3, rel_x
    assert torch.isfinite(xd.float()).all()


def test_stack_varies_selection_and_tau0_equals_dense(cuda):
    """The random-init stack selects different budgets per layer; at tau = 0
    every layer keeps all tokens and the stack equals the dense stack bitwise
    (test_model.cpp:226-243 at stack level)."""
    from paper_2602_03216_b200.stack import structured_hidden
    L = 2048
    st = _stack(L, n_layers=3)
    x = structured_hidden(L, 512, seed=2)
    st.forward(x.clone())
    kk = st.k_keep.cpu().tolist()
    assert all(1 <= k <= L for k in kk) and len(set(kk)) > 1, kk
    s0 = _stack(L, n_layers=2, tau=0.0)
    a = s0.forward(x.clone())
    assert s0.k_keep.cpu().tolist() == [L, L]
    b = s0.forward(x.clone(), dense=True)
    assert torch.equal(a.view(torch.int16), b.view(torch.int16))
    assert torch.isfinite(a.float()).all()


@pytest.mark.parametrize("rows,cols", [(40, 64), (129, 4096), (1, 3)])
def test_layer_drift_f32_bit_exact(cuda, port, rows, cols):
    """compute_drift (drift.cpp:14-45) per boundary: double sums in the
    reference's order -> bit-exact against the oracle (pinned to drift.cpp)."""
    rng = RefRng(rows * 7 + cols)
    h = np.stack([rng.random_matrix(rows, cols, 1.0 + 0.3 * i) for i in range(3)])
    ref = port.compute_drift(h, 1e-6)
    for l in range(2):
        g = float(tsa.layer_drift(dev(h[l]), dev(h[l + 1]), 1e-6).item())
        assert np.float64(g).view(np.uint64) == ref[l].view(np.uint64)


def test_select_sparse_layers_matches_oracle(cuda, port):
    for R in ([0.3, 0.1, 0.2, 0.4], [1.0, 1.0, 1.0], [0.5], [0.2, 0.2, 0.1, 0.3, 0.1]):
        for delta in (0.0, 0.25, 0.5, 1.0):
            rh, layers = tsa.select_sparse_layers(R, delta)
            orh, ol = port.select_sparse_layers(np.array(R), delta)
            assert np.array_equal(np.array(rh), orh) and layers == ol


def test_stack_drift_calibration_selects_half(cuda):
    """drift.cpp:67-80 on the stack: delta = 0.5 picks the lower-drift half of
    the layers; those run sparse, the rest dense (budget = L)."""
    from paper_2602_03216_b200.stack import structured_hidden
    L = 1024
    st = _stack(L, n_layers=4)
    x = structured_hidden(L, 512, seed=3)
    prof = st.calibrate(x, delta=0.5)
    assert len(prof["sparse_layers"]) == 2 and len(prof["R"]) == 4
    st.forward(x.clone())
    kk = st.k_keep.cpu().tolist()
    for i in range(4):
        if i in prof["sparse_layers"]:
            assert kk[i] <= L
        else:
            assert kk[i] == L


def test_report_harness_rows(cuda):
    """report.py: the reference's sweep / fixed-vs-dynamic rows (bench.cpp:275-314)
    with the measured columns, in its CSV layout."""
    import io
    from paper_2602_03216_b200 import report
    base = ["--n-layers", "4", "--n-heads", "8", "--n-kv-heads", "2", "--d-model", "512",
            "--reps", "1"]
    for cmd in (["sweep", "--seq-lens", "2048"], ["fixed-vs-dynamic", "--seq-len", "2048"]):
        buf = io.StringIO()
        import contextlib
        with contextlib.redirect_stdout(buf):
            assert report.main(cmd + base + ["--format", "csv"]) == 0
        lines = buf.getvalue().splitlines()
        assert lines[0].startswith("# config ") and lines[1].startswith("# reference ")
        hdr = lines[2].split(",")
        assert hdr[-3:] == ["ms", "dense_ms", "measured_speedup"] and "est_speedup" in hdr
        rows = [dict(zip(hdr, l.split(","))) for l in lines[3:]]
        assert len(rows) == (2 if cmd[0] == "sweep" else 4)
        for r in rows:
            assert float(r["ms"]) > 0 and float(r["est_speedup"]) >= 1.0
            assert 1 <= float(r["avg_k_keep"]) <= 2048


def test_stack_graphed_forward_equals_eager(cuda):
    """forward_graphed (one CUDA graph for the whole stack) == forward, bitwise, on
    the capturing call and on replays, with the per-layer budgets kept."""
    from paper_2602_03216_b200.stack import structured_hidden
    L = 2048
    st = _stack(L, n_layers=3)
    x0 = structured_hidden(L, 512, seed=6)
    ref = st.forward(x0.clone())
    kk_ref = st.k_keep.clone()
    x = torch.empty_like(x0)
    for _ in range(3):
        x.copy_(x0)
        st.forward_graphed(x)
        torch.cuda.synchronize()
        assert torch.equal(x.view(torch.int16), ref.view(torch.int16))
        assert torch.equal(st.k_keep, kk_ref)
