"""Pins the CPU oracle (oracle/tsa_oracle.c) before it is trusted as the
checker: against the reference compiled from /root/reference (bit-exact), the
reference-generated golden fixtures, and the reference tests' inline
known-answer tests (test_tensor_ops.cpp, test_coverage.cpp, test_attention.cpp).
CPU only."""
import math

import numpy as np
import pytest

from oracle.oracle import OracleError, RefRng, equiv_heads, gqa_heads, rel_l2
from tests.golden.make_golden import load_cases


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


# ------------------------------------------------------------ golden fixtures
@pytest.mark.parametrize("name", sorted(load_cases().keys()))
def test_port_matches_reference_golden(port, name):
    c = load_cases()[name]
    s = port.score_tokens(c["q"], c["k"], c["last_q"], c["kernel"])
    assert np.array_equal(bits(s), bits(c["scores"]))
    k_keep = port.coverage_budget(port.aggregate_scores(s), c["tau"], max(1, len(c["forced"])))
    assert k_keep == c["k_keep"]
    idx = port.select_tokens(s, k_keep, c["forced"])
    assert np.array_equal(idx, c["idx"])
    out = port.token_sparse_attention(c["q"], c["k"], c["v"], idx)
    assert np.array_equal(bits(out), bits(c["out"]))


# ----------------------------------------------- port vs compiled reference
@pytest.mark.parametrize("H,Hkv,L,d,lq,ker", [
    (4, 2, 96, 16, 32, 7), (8, 2, 300, 32, 64, 7), (2, 2, 12, 8, 500, 1),
    (4, 4, 128, 16, 64, 5), (1, 1, 1, 4, 64, 7), (2, 1, 5, 4, 3, 7), (3, 1, 257, 8, 64, 9)])
def test_port_bit_exact_vs_reference(port, ref, H, Hkv, L, d, lq, ker):
    rng = RefRng(1000 + L + H)
    q, k, v = gqa_heads(rng, H, Hkv, L, d)
    s1, s2 = port.score_tokens(q, k, lq, ker), ref.score_tokens(q, k, lq, ker)
    assert np.array_equal(bits(s1), bits(s2))
    a1, a2 = port.aggregate_scores(s1), ref.aggregate_scores(s2)
    assert np.array_equal(bits(a1), bits(a2))
    for tau in (0.0, 0.005, 0.1, 0.5, 0.99, 1.0):
        for f in ([L - 1], list(range(max(0, L - 4), L)), []):
            mk = max(1, len(f))
            k1, k2 = port.coverage_budget(a1, tau, mk), ref.coverage_budget(a2, tau, mk)
            assert k1 == k2
            i1, i2 = port.select_tokens(s1, k1, f), ref.select_tokens(s2, k2, f)
            assert np.array_equal(i1, i2)
        o1 = port.token_sparse_attention(q, k, v, i1)
        o2 = ref.token_sparse_attention(q, k, v, i2, f)
        assert np.array_equal(bits(o1), bits(o2))


def test_port_threads_bit_identical(port):
    rng = RefRng(5)
    q, k, v = gqa_heads(rng, 8, 2, 200, 16)
    s1 = port.score_tokens(q, k, 64, 7, n_threads=1)
    s8 = port.score_tokens(q, k, 64, 7, n_threads=8)
    assert np.array_equal(bits(s1), bits(s8))
    idx = port.select_tokens(s1, 120, [199])
    o1 = port.token_sparse_attention(q, k, v, idx, n_threads=1)
    o8 = port.token_sparse_attention(q, k, v, idx, n_threads=8)
    assert np.array_equal(bits(o1), bits(o8))


def test_sampled_rows_equal_full(port):
    rng = RefRng(6)
    q, k, v = gqa_heads(rng, 4, 2, 160, 16)
    idx = port.select_tokens(port.score_tokens(q, k, 64, 7), 100, [159])
    full = port.token_sparse_attention(q, k, v, idx)
    samp = port.token_sparse_attention_sampled(q, k, v, idx, head_stride=2, r0=10, r1=60)
    for h in (0, 2):
        rows = idx[h, 10:60]
        assert np.array_equal(bits(samp[h, rows]), bits(full[h, rows]))


def test_reference_prefix_sample_matches_full(port, ref):
    rng = RefRng(8)
    q, k, v = gqa_heads(rng, 4, 2, 128, 16)
    idx = port.select_tokens(port.score_tokens(q, k, 64, 7), 90, [127])
    full = port.token_sparse_attention(q, k, v, idx)
    pre = ref.tsa_head_prefix(q, k, v, idx, h=3, m=40)
    assert np.array_equal(bits(pre), bits(full[3, idx[3, :40]]))


def test_run_equiv_grid_subset_meets_gate(port):
    """run_equiv (bench.cpp:225-273): fast path vs masked_sparse_oracle <= 1e-5."""
    grid = [(L, H, d, tau) for L in (16, 64, 256) for H in (1, 4, 8) for d in (8, 16, 32)
            for tau in (0.0, 0.005, 0.1, 0.5, 0.99)]
    for i in range(0, len(grid), 9):
        L, H, d, tau = grid[i]
        q, k, v = equiv_heads(42, i, L, H, d)
        s = port.score_tokens(q, k, 64, 7)
        kk = port.coverage_budget(port.aggregate_scores(s), tau, 1)
        idx = port.select_tokens(s, kk, [L - 1])
        fast = port.token_sparse_attention(q, k, v, idx)
        err = max(np.abs(fast[h] - port.masked_sparse_oracle(q[h], k[h], v[h], idx[h])).max()
                  for h in range(H))
        assert err <= 1e-5
        if tau == 0.0:  # test_bench.cpp:134-145
            assert kk == L and err == 0.0


# ------------------------------------------- reference inline KATs (restated)
def test_kat_score_d1(port):
    # test_coverage.cpp:54-71
    q = np.array([[[1.0], [1.0]]], np.float32)
    k = np.array([[[0.0], [math.log(3.0)]]], np.float32)
    s = port.score_tokens(q, k, 1, 1)
    assert s.shape == (1, 2)
    assert abs(s[0, 0] - 0.25) < 1e-6 and abs(s[0, 1] - 0.75) < 1e-6


def test_kat_kernel1_mass(port):
    # test_coverage.cpp:73-87
    rng = RefRng(30)
    for L in (8, 64, 200):
        for lq in (1, 16, 1000):
            q, k, _ = gqa_heads(rng, 4, 2, L, 16)
            s = port.score_tokens(q, k, lq, 1)
            np.testing.assert_allclose(s.astype(np.float64).sum(1), min(lq, L), rtol=1e-6)


def test_kat_aggregate_and_zero(port):
    # test_coverage.cpp:136-151
    sl = port.aggregate_scores(np.array([[1, 2, 1], [3, 0, 1]], np.float32))
    np.testing.assert_allclose(sl, [0.5, 0.25, 0.25], rtol=1e-6)
    with pytest.raises(OracleError, match="all scores are zero"):
        port.aggregate_scores(np.zeros((2, 2), np.float32))


def test_kat_coverage_budget(port):
    # test_coverage.cpp:155-208
    a = np.array([0.4, 0.3, 0.2, 0.1], np.float32)
    assert port.coverage_budget(a, 0.25, 1) == 2
    assert port.coverage_budget(a, 0.0, 1) == 4
    assert port.coverage_budget(a, 1.0, 1) == 1 and port.coverage_budget(a, 1.0, 3) == 3
    u = np.full(4, 0.25, np.float32)
    assert [port.coverage_budget(u, t, 1) for t in (0.5, 0.26, 0.24)] == [2, 2, 3]
    m = np.array([0.7, 0.1, 0.1, 0.1], np.float32)
    assert port.coverage_budget(m, 0.9, 1) == 1 and port.coverage_budget(m, 0.9, 2) == 2
    for bad in ((-0.1, 1), (1.1, 1), (0.5, 0), (0.5, 5)):
        with pytest.raises(OracleError):
            port.coverage_budget(a, *bad)


def test_kat_fixed_budget(port):
    # test_coverage.cpp:212-223
    assert port.fixed_budget(1000, 0.3) == 700 and port.fixed_budget(1000, 0.5) == 500
    assert port.fixed_budget(256, 0.5) == 128 and port.fixed_budget(10, 0.95) == 1
    assert port.fixed_budget(10, 0.95, 4) == 4
    for bad in (-0.1, 1.0):
        with pytest.raises(OracleError):
            port.fixed_budget(100, bad)


def test_kat_select_tokens(port):
    # test_coverage.cpp:227-296
    s = np.array([[0.1, 0.9, 0.3, 0.5], [0.8, 0.1, 0.7, 0.2]], np.float32)
    assert port.select_tokens(s, 2).tolist() == [[1, 3], [0, 2]]
    assert port.select_tokens(np.full((1, 4), 0.5, np.float32), 2).tolist() == [[0, 1]]
    f = np.array([[0.9, 0.8, 0.7, 0.01]], np.float32)
    assert port.select_tokens(f, 2, [3]).tolist() == [[0, 3]]
    assert port.select_tokens(f, 1, [3]).tolist() == [[3]]
    r = np.array([[0.1, 0.2, 0.3, 0.4]], np.float32)
    assert port.select_tokens(r, 2, [1, 0]).tolist() == [[0, 1]]
    assert port.select_tokens(r, 2, [1, 1]).tolist() == [[1, 3]]
    for k_keep, forced in ((0, []), (5, []), (1, [0, 1]), (2, [4])):
        with pytest.raises(OracleError):
            port.select_tokens(r, k_keep, forced)


def test_kat_attention(port):
    # test_attention.cpp:126-158, 180-200
    v = np.array([[3.0, -1.0]], np.float32)
    assert np.array_equal(port.dense_causal_attention(np.zeros((1, 2), np.float32),
                                                      np.zeros((1, 2), np.float32), v), v)
    n, d = 6, 3
    vv = RefRng(1).random_matrix(n, d)
    o = port.dense_causal_attention(np.zeros((n, d), np.float32), np.zeros((n, d), np.float32), vv)
    for t in range(n):
        np.testing.assert_allclose(o[t], vv[: t + 1].astype(np.float64).mean(0), rtol=1e-6,
                                   atol=1e-7)
    q = RefRng(2).random_matrix(2, 4)
    kk = RefRng(3).random_matrix(2, 4)
    v2 = RefRng(4).random_matrix(2, 4)
    o = port.masked_sparse_oracle(q, kk, v2, [0])
    assert np.array_equal(o[0], v2[0]) and np.all(o[1] == 0.0)


def test_rel_l2_metric():
    # bench.cpp:199-214
    a = np.array([[1.0, 2.0]], np.float32)
    assert rel_l2(a, a) == 0.0
    assert abs(rel_l2(np.array([[1.0, 0.0]]), np.array([[0.0, 0.0]])) - 1.0) < 1e-12


# ------------------------------------- attention-branch producer (model.cpp)
def test_producer_port_bit_exact_vs_reference(port, ref):
    """rms_norm / apply_rope / project_qkv: the C restatement against the
    reference's model.cpp compiled from /root/reference."""
    rng = RefRng(31)
    x = rng.random_matrix(37, 96, 2.0)
    g = rng.random_matrix(1, 96, 1.0).reshape(-1)
    for eps in (0.0, 1e-5):
        assert np.array_equal(bits(port.rms_norm(x, g, eps)), bits(ref.rms_norm(x, g, eps)))
    y = rng.random_matrix(300, 64, 1.0)
    for theta in (10000.0, 500000.0):
        assert np.array_equal(bits(port.apply_rope(y, theta)), bits(ref.apply_rope(y, theta)))
    xn = rng.random_matrix(50, 64, 1.0)
    wq, wk, wv = (rng.random_matrix(64, w, 0.2) for w in (4 * 16, 2 * 16, 2 * 16))
    a = port.project_qkv(xn, wq, wk, wv, 4, 2, 16, 10000.0)
    b = ref.project_qkv(xn, wq, wk, wv, 4, 2, 16, 10000.0)
    for p, r in zip(a, b):
        assert np.array_equal(bits(p), bits(r))


def test_producer_kats(port):
    """test_model.cpp:75-155: unit-gain rows have unit RMS; gain scales columns;
    eps keeps zero rows finite; position 0 is the identity; rotation preserves
    pair norms; q.k depends only on the relative position; odd widths throw."""
    rng = RefRng(32)
    x = rng.random_matrix(3, 16, 3.0)
    y = port.rms_norm(x, np.ones(16, np.float32), 0.0)
    assert np.allclose(np.sqrt((y.astype(np.float64) ** 2).mean(axis=1)), 1.0, atol=1e-6)
    g = np.arange(1, 17, dtype=np.float32)
    assert np.allclose(port.rms_norm(x, g, 0.0), y * g, rtol=1e-6)
    assert np.all(np.isfinite(port.rms_norm(np.zeros((2, 4), np.float32), np.ones(4, np.float32),
                                            1e-5)))
    r = rng.random_matrix(64, 8, 1.0)
    ro = port.apply_rope(r, 10000.0)
    assert np.array_equal(bits(ro[0]), bits(r[0]))
    n0 = np.hypot(r[:, 0::2], r[:, 1::2])
    assert np.allclose(np.hypot(ro[:, 0::2], ro[:, 1::2]), n0, rtol=1e-5)
    q = np.tile(rng.random_matrix(1, 8, 1.0), (64, 1))
    k = np.tile(rng.random_matrix(1, 8, 1.0), (64, 1))
    rq, rk = port.apply_rope(q, 10000.0), port.apply_rope(k, 10000.0)
    d1 = float(rq[20] @ rk[15])   # relative offset 5
    d2 = float(rq[40] @ rk[35])
    assert abs(d1 - d2) < 1e-4 * max(1.0, abs(d1))
    with pytest.raises(OracleError):
        port.apply_rope(np.zeros((1, 3), np.float32), 1e4)


def test_report_flop_model_matches_reference(ref):
    """paper_2602_03216_b200.report.estimate_flops restates flops.cpp:12-51: the
    same doubles as the reference compiled here."""
    from paper_2602_03216_b200.report import estimate_flops
    cases = [(131072, 128, 32, [75533] * 16 + [None] * 16),
             (4096, 16, 8, [2027, None, 1, 4096]), (256, 8, 1, [None]), (100, 4, 2, [50])]
    for L, d, H, kk in cases:
        for lq, ker in ((64, 7), (500, 1)):
            a = estimate_flops(L, d, H, kk, lq, ker)
            b = ref.estimate_flops(L, d, H, kk, lq, ker)
            for key, v in b.items():
                assert a[key] == v, (key, a[key], v)


def test_drift_port_bit_exact_vs_reference(port, ref):
    rng = RefRng(41)
    h = np.stack([rng.random_matrix(33, 48, 1.0 + 0.2 * i) for i in range(4)])
    a, b = port.compute_drift(h, 1e-6), ref.compute_drift(h, 1e-6)
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
    for delta in (0.0, 0.5, 1.0):
        pa, pb = port.select_sparse_layers(a, delta), ref.select_sparse_layers(b, delta)
        assert np.array_equal(pa[0], pb[0]) and pa[1] == pb[1]
