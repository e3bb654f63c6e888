"""Parity of the CUDA path (through the C ABI) against the CPU oracle and the
reference-generated golden fixtures.  Runs on the B200 box: -m gpu."""
import numpy as np
import pytest
import torch

import paper_2602_03216_b200 as tsa
from oracle.oracle import RefRng, equiv_heads, gqa_heads
from tests import parity
from tests.golden.make_golden import load_cases

pytestmark = pytest.mark.gpu

CASES = load_cases()


def dev(a, dtype=torch.float32):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dtype)


def host(t):
    return t.detach().float().cpu().numpy()


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def heads_of(q, k, v, dtype=torch.float32):
    return tsa.HeadTensors(dev(q, dtype), dev(k, dtype), dev(v, dtype))


# ------------------------------------------------------------------ scoring
@pytest.mark.parametrize("name", sorted(CASES))
def test_score_reference_mode_vs_golden(cuda, name):
    c = CASES[name]
    hs = tsa.score_tokens(heads_of(c["q"], c["k"], c["v"]), c["last_q"], c["kernel"])
    s = host(hs.s)
    exact = np.mean(bits(s) == bits(c["scores"]))
    assert exact >= 0.99, f"only {exact:.4f} of scores bit-identical"
    np.testing.assert_allclose(s, c["scores"], rtol=4 * 2**-23, atol=1e-30)


def test_score_bf16_inputs_match_oracle_on_upcast(cuda, port):
    q, k, v = gqa_heads(RefRng(11), 8, 2, 1000, 128)
    hq = heads_of(q, k, v, torch.bfloat16)
    up = [host(t) for t in (hq.q, hq.k)]
    s_gpu = host(tsa.score_tokens(hq, 64, 7, scoring=1).s)
    s_ora = port.score_tokens(up[0], up[1], 64, 7)
    assert np.mean(bits(s_gpu) == bits(s_ora)) >= 0.99


# ----------------------------------------------------- budget / selection
@pytest.mark.parametrize("name", sorted(CASES))
def test_budget_and_select_on_oracle_scores_bit_exact(cuda, port, name):
    """Integer stages fed identical scores must agree exactly."""
    c = CASES[name]
    s = dev(c["scores"])
    sl = tsa.aggregate_scores(tsa.HeadScores(s))
    assert np.array_equal(bits(host(sl.s)), bits(port.aggregate_scores(c["scores"])))
    k_gpu = tsa.coverage_budget(sl, c["tau"], max(1, len(c["forced"])))
    k_ora, pp, pa = port.coverage_budget(host(sl.s), c["tau"], max(1, len(c["forced"])),
                                         with_prefix=True)
    parity.check_budget(k_gpu, k_ora, pp, pa, c["tau"], c["L"])
    assert k_ora == c["k_keep"]
    sel = tsa.select_tokens(tsa.HeadScores(s), c["k_keep"], c["forced"])
    assert np.array_equal(host(sel.indices).astype(np.int32), c["idx"])


@pytest.mark.parametrize("L,H,tau,seed", [(4096, 8, 0.005, 1), (4096, 8, 0.1, 2),
                                          (4096, 8, 0.5, 3), (2000, 4, 0.99, 4),
                                          (131072, 2, 0.01, 5), (65537, 4, 0.3, 6),
                                          (150001, 2, 0.01, 7)])  # slice > 16384: global path
def test_budget_random_scores(cuda, port, L, H, tau, seed):
    rng = np.random.default_rng(seed)
    # heavy-tailed positive scores with ties
    s = np.exp(rng.normal(0, 3, (H, L))).astype(np.float32)
    s[:, ::17] = s[:, 3:4]
    s_dev = dev(s)
    k_gpu = tsa.coverage_budget(tsa.aggregate_scores(tsa.HeadScores(s_dev)), tau, 1)
    sl = port.aggregate_scores(s)
    k_ora, pp, pa = port.coverage_budget(sl, tau, 1, with_prefix=True)
    parity.check_budget(k_gpu, k_ora, pp, pa, tau, L)


@pytest.mark.parametrize("L,k,nf", [(1, 1, 1), (10, 3, 1), (4096, 1000, 1), (4096, 4096, 1),
                                    (5000, 64, 64), (131072, 70000, 1), (3000, 1, 1),
                                    (150001, 80000, 1), (140000, 140000, 64)])
def test_select_random_with_ties(cuda, port, L, k, nf):
    rng = np.random.default_rng(L + k)
    s = rng.integers(0, 50, (4, L)).astype(np.float32) / 7.0  # many exact ties
    forced = list(range(L - nf, L))
    sel = tsa.select_tokens(tsa.HeadScores(dev(s)), k, forced)
    assert np.array_equal(host(sel.indices).astype(np.int32), port.select_tokens(s, k, forced))


def test_select_kats(cuda):
    # test_coverage.cpp:227-296
    def sel(rows, k, forced=()):
        return host(tsa.select_tokens(tsa.HeadScores(dev(np.array(rows, np.float32))), k,
                                      forced).indices).astype(int).tolist()
    assert sel([[0.1, 0.9, 0.3, 0.5], [0.8, 0.1, 0.7, 0.2]], 2) == [[1, 3], [0, 2]]
    assert sel([[0.5, 0.5, 0.5, 0.5]], 2) == [[0, 1]]
    assert sel([[0.9, 0.8, 0.7, 0.01]], 2, [3]) == [[0, 3]]
    assert sel([[0.9, 0.8, 0.7, 0.01]], 1, [3]) == [[3]]
    assert sel([[0.1, 0.2, 0.3, 0.4]], 2, [1, 0]) == [[0, 1]]
    assert sel([[0.1, 0.2, 0.3, 0.4]], 2, [1, 1]) == [[1, 3]]
    with pytest.raises(tsa.InvalidArgument):
        sel([[0.1, 0.2, 0.3, 0.4]], 1, [0, 1])
    with pytest.raises(tsa.InvalidArgument):
        sel([[0.1, 0.2, 0.3, 0.4]], 5)


def test_budget_kats(cuda):
    def cb(v, tau, mk=1):
        return tsa.coverage_budget(tsa.LayerScores(dev(np.array(v, np.float32))), tau, mk)
    a = [0.4, 0.3, 0.2, 0.1]
    assert cb(a, 0.25) == 2 and cb(a, 0.0) == 4 and cb(a, 1.0) == 1 and cb(a, 1.0, 3) == 3
    assert [cb([0.25] * 4, t) for t in (0.5, 0.26, 0.24)] == [2, 2, 3]
    assert cb([0.7, 0.1, 0.1, 0.1], 0.9) == 1 and cb([0.7, 0.1, 0.1, 0.1], 0.9, 2) == 2
    with pytest.raises(tsa.InvalidArgument):
        tsa.aggregate_scores(tsa.HeadScores(dev(np.zeros((2, 2), np.float32))))


# ---------------------------------------------------------------- attention
@pytest.mark.parametrize("name", sorted(CASES))
def test_token_sparse_attention_vs_golden(cuda, name):
    c = CASES[name]
    h = heads_of(c["q"], c["k"], c["v"])
    sel = tsa.TokenSelection(indices=dev(c["idx"], torch.int32), k_keep=c["k_keep"],
                             forced=c["forced"])
    out = host(tsa.token_sparse_attention(h, sel))
    assert np.abs(out - c["out"]).max() <= parity.F32_GATE
    assert parity.unselected_rows_zero(out, c["idx"], c["L"])


@pytest.mark.parametrize("name", sorted(CASES))
def test_sparse_layer_end_to_end_vs_golden(cuda, port, name):
    c = CASES[name]
    plan = tsa.SparsePlan(mode=tsa.SparseMode.kDynamic, sparse_layers=[0], tau=c["tau"],
                          last_q=c["last_q"], kernel=c["kernel"],
                          forced=tsa.ForcedPolicy(c["policy"]))
    out, st = tsa.sparse_attention_layer(heads_of(c["q"], c["k"], c["v"]), plan)
    assert st.k_keep == c["k_keep"]
    idx = host(st.selection.indices).astype(np.int32)
    parity.check_index_sets(idx, c["idx"], c["scores"], c["forced"])
    if np.array_equal(idx, c["idx"]):
        assert np.abs(host(out) - c["out"]).max() <= parity.F32_GATE


def test_run_equiv_full_grid(cuda, port):
    """All 135 run_equiv instances (bench.cpp:225-273) through the GPU layer
    call, checked against masked_sparse_oracle at the 1e-5 gate."""
    grid = [(L, H, d, tau) for L in (16, 64, 256) for H in (1, 4, 8) for d in (8, 16, 32)
            for tau in (0.0, 0.005, 0.1, 0.5, 0.99)]
    for i, (L, H, d, tau) in enumerate(grid):
        q, k, v = equiv_heads(42, i, L, H, d)
        plan = tsa.SparsePlan(mode=tsa.SparseMode.kDynamic, sparse_layers=[0], tau=tau)
        out, st = tsa.sparse_attention_layer(heads_of(q, k, v), plan)
        idx = host(st.selection.indices).astype(np.int32)
        o = host(out)
        err = max(np.abs(o[h] - port.masked_sparse_oracle(q[h], k[h], v[h], idx[h])).max()
                  for h in range(H))
        assert err <= parity.F32_GATE, (i, L, H, d, tau, err)
        if tau == 0.0:
            assert st.k_keep == L


@pytest.mark.parametrize("H,Hkv,L,n", [(4, 2, 128, 128), (4, 2, 300, 300), (2, 1, 1000, 777),
                                       (8, 8, 2048, 2048), (4, 1, 4096, 1500), (2, 2, 129, 1)])
def test_tcgen05_attention_bf16_vs_oracle(cuda, port, H, Hkv, L, n):
    q, k, v = gqa_heads(RefRng(L + n), H, Hkv, L, 128)
    h = heads_of(q, k, v, torch.bfloat16)
    up = [host(t) for t in (h.q, h.k, h.v)]
    rng = np.random.default_rng(n)
    idx = np.stack([np.sort(rng.choice(L, n, replace=False)) for _ in range(H)]).astype(np.int32)
    sel = tsa.TokenSelection(indices=dev(idx, torch.int32), k_keep=n, forced=[])
    out = host(tsa.token_sparse_attention(h, sel))
    ref = port.token_sparse_attention(up[0], up[1], up[2], idx, n_threads=8)
    assert parity.rel_l2(out, ref) <= parity.BF16_REL_L2
    assert parity.unselected_rows_zero(out, idx, L)


@pytest.mark.parametrize("H,Hkv,L", [(4, 2, 512), (2, 1, 1000), (4, 4, 2048)])
def test_dense_attention_bf16_and_f32(cuda, port, H, Hkv, L):
    q, k, v = gqa_heads(RefRng(L), H, Hkv, L, 128)
    for dt, gate in ((torch.bfloat16, "bf16"), (torch.float32, "f32")):
        h = heads_of(q, k, v, dt)
        up = [host(t) for t in (h.q, h.k, h.v)]
        out = torch.empty_like(h.q)
        for i in range(H):
            out[i] = tsa.dense_causal_attention(h.q[i], h.k[h.kv_head(i)], h.v[h.kv_head(i)])
        for i in (0, H - 1):
            ref = port.dense_causal_attention(up[0][i], up[1][i * Hkv // H], up[2][i * Hkv // H])
            o = host(out[i])
            if gate == "bf16":
                assert parity.rel_l2(o, ref) <= parity.BF16_REL_L2
            else:
                assert np.abs(o - ref).max() <= parity.F32_GATE


def test_tau0_equals_dense_bitwise(cuda):
    """test_bench.cpp:134-145 / SPEC: tau = 0 keeps every token and the sparse
    path reproduces dense attention exactly (same kernel, same inputs)."""
    q, k, v = gqa_heads(RefRng(21), 4, 2, 640, 128)
    for dt in (torch.bfloat16, torch.float32):
        h = heads_of(q, k, v, dt)
        plan = tsa.SparsePlan(mode=tsa.SparseMode.kDynamic, sparse_layers=[0], tau=0.0)
        out, st = tsa.sparse_attention_layer(h, plan)
        dense, _ = tsa.sparse_attention_layer(h, tsa.SparsePlan())
        assert st.k_keep == 640
        assert torch.equal(out, dense)


@pytest.mark.parametrize("L", [640, 3000])
def test_tau0_reads_kv_in_place(cuda, L):
    """k_keep == L: the selection is the identity, the fused pair skips the
    compressed K/V copy and the attention reads the KV heads in place -- the
    output equals dense attention bitwise through every entry point, and the
    compressed buffers are not read (poisoned with NaN here)."""
    from paper_2602_03216_b200 import workloads
    from paper_2602_03216_b200.dist import ShardedSparseAttention
    q, k, v = workloads.heavy_tailed_heads(8, 2, L, 128, seed=31)
    plan = tsa.SparsePlan(mode=tsa.SparseMode.kDynamic, sparse_layers=[0], tau=0.0)
    dense, _ = tsa.sparse_attention_layer(tsa.HeadTensors(q, k, v), tsa.SparsePlan())
    lay = ShardedSparseAttention(8, 2, L, 128, torch.bfloat16, plan, device=q.device)
    lay.backend.kc.fill_(float("nan"))
    lay.backend.vc.fill_(float("nan"))
    o = lay.step(q, k, v)
    torch.cuda.synchronize()
    assert lay.k_keep == L
    assert torch.equal(o.view(torch.int16), dense.view(torch.int16))
    assert bool(torch.isnan(lay.backend.kc).all())  # the copy was skipped
    hq, hk, hv = (t.cpu().pin_memory() for t in (q, k, v))
    hout = torch.empty(q.shape, dtype=q.dtype).pin_memory()
    tsa.sparse_attention_layer_host(hq, hk, hv, hout, plan, n_groups=2)
    torch.cuda.synchronize()
    assert torch.equal(hout.view(torch.int16), dense.cpu().view(torch.int16))
    # one token short of L: the compressed path again, still causal-exact
    plan_f = tsa.SparsePlan(mode=tsa.SparseMode.kFixed, sparse_layers=[0], s_fixed=1.0 / L)
    out_f, st_f = tsa.sparse_attention_layer(tsa.HeadTensors(q, k, v), plan_f)
    assert st_f.k_keep == L - 1


def test_kv_tiles_never_read_the_next_head(cuda):
    """L % 128 != 0: the last K/V tile of a head runs past its rows.  Those keys
    are masked, but P = 0 times a NaN would still poison O, so in the indexed
    (production) kernel the V tile reads zeros there, not the next KV head's
    rows -- the host-tensor pipeline copies V per head group, so the next
    head's rows may not have arrived yet.  NaN in KV head 1 must leave the
    outputs of KV head 0's query heads bitwise unchanged on the in-place
    (k_keep = L) path.  (The dense baseline kernel reads the next head's rows
    there -- the caller's finite data, masked.)"""
    from paper_2602_03216_b200 import workloads
    from paper_2602_03216_b200.dist import ShardedSparseAttention
    L = 3000
    q, k, v = workloads.heavy_tailed_heads(8, 2, L, 128, seed=33)
    v_nan = v.clone()
    v_nan[1, :72] = float("nan")
    k_nan = k.clone()
    k_nan[1, :72] = float("nan")
    clean, _ = tsa.sparse_attention_layer(tsa.HeadTensors(q, k, v), tsa.SparsePlan())
    plan = tsa.SparsePlan(mode=tsa.SparseMode.kDynamic, sparse_layers=[0], tau=0.0)
    lay = ShardedSparseAttention(8, 2, L, 128, torch.bfloat16, plan, device=q.device)
    b = lay.backend
    lay.step(q, k, v)  # identity selection
    assert lay.k_keep == L
    out = torch.empty_like(q)
    b.attend_indexed(q, k_nan, v_nan, b.k_keep, out)
    torch.cuda.synchronize()
    assert torch.equal(out[:4].view(torch.int16), clean[:4].view(torch.int16))


def test_causality_bitwise(cuda):
    """test_attention.cpp:293-316: perturbing K/V after row t leaves rows <= t unchanged."""
    q, k, v = gqa_heads(RefRng(22), 4, 2, 512, 128)
    for dt in (torch.bfloat16, torch.float32):
        h = heads_of(q, k, v, dt)
        plan = tsa.SparsePlan(mode=tsa.SparseMode.kFixed, sparse_layers=[0], s_fixed=0.5)
        base, st = tsa.sparse_attention_layer(h, plan)
        sel = st.selection
        cut = 300
        k2, v2 = h.k.clone(), h.v.clone()
        k2[:, cut + 1:] += 3.0
        v2[:, cut + 1:] -= 2.0
        pert = tsa.token_sparse_attention(tsa.HeadTensors(h.q, k2, v2), sel)
        assert torch.equal(base[:, : cut + 1], pert[:, : cut + 1])


def test_inner_seam_sees_compressed_shapes(cuda):
    """test_attention.cpp:318-338: `inner` is called once per head with k x d."""
    q, k, v = gqa_heads(RefRng(23), 4, 2, 100, 16)
    h = heads_of(q, k, v)
    sel = tsa.select_tokens(tsa.score_tokens(h, 64, 7), 37, [99])
    shapes = []

    def probe(qc, kc, vc):
        shapes.append((tuple(qc.shape), tuple(kc.shape), tuple(vc.shape)))
        return tsa.dense_causal_attention(qc, kc, vc)

    a = tsa.token_sparse_attention(h, sel, inner=probe)
    b = tsa.token_sparse_attention(h, sel)
    assert shapes == [((37, 16),) * 3] * 4
    assert torch.equal(a, b)


def test_fixed_mode_and_recent_window(cuda, port):
    q, k, v = gqa_heads(RefRng(24), 8, 2, 700, 32)
    h = heads_of(q, k, v)
    plan = tsa.SparsePlan(mode=tsa.SparseMode.kFixed, sparse_layers=[0], s_fixed=0.3,
                          forced=tsa.ForcedPolicy.kRecentWindow, last_q=50)
    out, st = tsa.sparse_attention_layer(h, plan)
    assert st.k_keep == port.fixed_budget(700, 0.3, 50) == 490
    s = port.score_tokens(q, k, 50, 7)
    forced = list(range(650, 700))
    ora_idx = port.select_tokens(s, 490, forced)
    idx = host(st.selection.indices).astype(np.int32)
    parity.check_index_sets(idx, ora_idx, s, forced)
    ref = port.token_sparse_attention(q, k, v, idx)
    assert np.abs(host(out) - ref).max() <= parity.F32_GATE


def test_dense_layer_not_in_plan(cuda):
    q, k, v = gqa_heads(RefRng(25), 4, 2, 256, 128)
    h = heads_of(q, k, v, torch.bfloat16)
    plan = tsa.SparsePlan(mode=tsa.SparseMode.kDynamic, sparse_layers=[1], tau=0.5)
    out, st = tsa.sparse_attention_layer(h, plan, layer=0)
    assert not st.sparse and st.k_keep == 256 and st.selection is None


def test_edge_lengths(cuda, port):
    for L in (1, 2, 3, 17):
        q, k, v = gqa_heads(RefRng(30 + L), 2, 1, L, 8)
        plan = tsa.SparsePlan(mode=tsa.SparseMode.kDynamic, sparse_layers=[0], tau=0.5)
        out, st = tsa.sparse_attention_layer(heads_of(q, k, v), plan)
        s = port.score_tokens(q, k, 64, 7)
        k_ora = port.coverage_budget(port.aggregate_scores(s), 0.5, 1)
        assert st.k_keep == k_ora
        idx = port.select_tokens(s, k_ora, [L - 1])
        assert np.array_equal(host(st.selection.indices).astype(np.int32), idx)
        assert np.abs(host(out) - port.token_sparse_attention(q, k, v, idx)).max() <= 1e-5


@pytest.mark.slow
def test_cfg1_full_size_f32(cuda, port):
    """BASELINE configs[0]: H=32/8, d=128, L=4096, f32, tau=0.5 vs the oracle."""
    rng = RefRng(2026)
    q, k, v = gqa_heads(rng, 32, 8, 4096, 128)
    h = heads_of(q, k, v)
    plan = tsa.SparsePlan(mode=tsa.SparseMode.kDynamic, sparse_layers=[0], tau=0.5)
    out, st = tsa.sparse_attention_layer(h, plan)
    s = port.score_tokens(q, k, 64, 7, n_threads=8)
    k_ora, pp, pa = port.coverage_budget(port.aggregate_scores(s), 0.5, 1, with_prefix=True)
    parity.check_budget(st.k_keep, k_ora, pp, pa, 0.5, 4096)
    idx = host(st.selection.indices).astype(np.int32)
    if st.k_keep == k_ora:
        parity.check_index_sets(idx, port.select_tokens(s, k_ora, [4095]), s, [4095])
    ref = port.token_sparse_attention_sampled(q, k, v, idx, head_stride=4, r0=0,
                                              r1=st.k_keep, n_threads=8)
    o = host(out)
    for hh in range(0, 32, 4):
        assert np.abs(o[hh] - ref[hh]).max() <= parity.F32_GATE


# -------------------------------------------------------------- FAST scoring
@pytest.mark.parametrize("H,Hkv,L,lq", [(8, 2, 4096, 64), (4, 4, 1000, 64), (8, 1, 3000, 32),
                                        (4, 2, 700, 128), (2, 2, 64, 64), (32, 8, 16384, 64)])
def test_score_fast_tensor_core_vs_oracle(cuda, port, H, Hkv, L, lq):
    from paper_2602_03216_b200 import workloads
    q, k, v = workloads.heavy_tailed_heads(H, Hkv, L, 128, sigma=3.0, seed=L, last_q=lq)
    h = tsa.HeadTensors(q, k, v)
    s_fast = host(tsa.score_tokens(h, lq, 7, scoring=2).s)
    up = [host(t) for t in (q, k)]
    s_ora = port.score_tokens(up[0], up[1], lq, 7, n_threads=8)
    # mass conservation (kernel 1 would be exact): per head ~ lq
    np.testing.assert_allclose(s_fast.astype(np.float64).sum(1), s_ora.astype(np.float64).sum(1),
                               rtol=1e-4)
    big = s_ora > 1e-6 * s_ora.max()
    rel = np.abs(s_fast - s_ora)[big] / s_ora[big]
    assert rel.max() <= parity.FAST_SCORE_REL, rel.max()
    tau = 0.01
    sl_o = port.aggregate_scores(s_ora)
    k_o, pp, pa = port.coverage_budget(sl_o, tau, 1, with_prefix=True)
    k_g = tsa.coverage_budget(tsa.aggregate_scores(tsa.HeadScores(dev(s_fast))), tau, 1)
    assert abs(k_g - k_o) <= max(2, int(parity.FAST_BUDGET_REL * L)), (k_g, k_o)
    sel_g = host(tsa.select_tokens(tsa.HeadScores(dev(s_fast)), k_o, [L - 1]).indices)
    parity.check_index_sets(sel_g.astype(np.int32), port.select_tokens(s_ora, k_o, [L - 1]),
                            s_ora, [L - 1], rel_tol=parity.FAST_SCORE_REL)


def test_reference_scoring_is_default_and_fast_deterministic(cuda):
    """DEFAULT scoring is the reference's arithmetic (bit-exact scores) for bf16
    too; FAST runs only on request and is deterministic."""
    from paper_2602_03216_b200 import workloads
    q, k, v = workloads.heavy_tailed_heads(8, 2, 8192, 128, seed=3)
    h = tsa.HeadTensors(q, k, v)
    a = tsa.score_tokens(h, 64, 7).s
    r = tsa.score_tokens(h, 64, 7, scoring=1).s
    b = tsa.score_tokens(h, 64, 7, scoring=2).s
    c = tsa.score_tokens(h, 64, 7, scoring=2).s
    assert torch.equal(a, r) and torch.equal(b, c) and not torch.equal(a, b)


def test_tcgen05_attention_running_max_rescales(cuda, port):
    """Keys whose logits grow along the sequence force the lazy O rescale on
    every KV tile for some rows but not others (warp-divergent decision)."""
    L, d = 1536, 128
    rng = np.random.default_rng(0)
    u = rng.normal(size=d)
    u /= np.linalg.norm(u)
    q = np.empty((2, L, d), np.float32)
    q[0] = np.sqrt(d) * u + 0.1 * rng.normal(size=(L, d))
    q[1] = rng.uniform(-1, 1, (L, d))            # a head that never rescales
    c = (np.arange(L) / 8.0)[:, None]             # +16 per 128-key tile
    k = (c * u[None, :] * np.where(np.arange(L) % 3 == 0, 1.0, -0.5)[:, None]
         + 0.1 * rng.normal(size=(L, d)))[None].astype(np.float32)
    v = rng.uniform(-1, 1, (1, L, d)).astype(np.float32)
    h = heads_of(q, k, v, torch.bfloat16)
    up = [host(t) for t in (h.q, h.k, h.v)]
    out = torch.empty_like(h.q)
    for i in range(2):
        out[i] = tsa.dense_causal_attention(h.q[i], h.k[0], h.v[0])
    for i in range(2):
        ref = port.dense_causal_attention(up[0][i], up[1][0], up[2][0])
        assert parity.rel_l2(host(out[i]), ref) <= parity.BF16_REL_L2


@pytest.mark.parametrize("indexed", [False, True])
def test_tcgen05_attention_all_logits_very_negative(cuda, indexed):
    """Every logit ~ -1100 (K = -Q, |q.k| large): softmax is shift-invariant, so
    each row is the mean of its causal V prefix (test_attention.cpp:126-158's
    Q = K = 0 case, shifted).  Guards the row max: a max that is not exactly
    the largest unmasked logit (e.g. an extra 0 or stale column) underflows
    every exponential and divides 0 by 0."""
    H, L, d = 2, 384, 128
    rng = np.random.default_rng(3)
    u = np.where(rng.uniform(size=d) < 0.5, -1.0, 1.0)
    q = np.broadcast_to(3.0 * u, (H, L, d)).astype(np.float32)
    k = np.broadcast_to(-3.0 * u, (1, L, d)).astype(np.float32)
    v = rng.uniform(-1, 1, (1, L, d)).astype(np.float32)
    h = heads_of(q, k, v, torch.bfloat16)
    vv = host(h.v)[0].astype(np.float64)
    ref = np.cumsum(vv, axis=0) / np.arange(1, L + 1)[:, None]
    if indexed:  # the fused path at tau = 0 (every token kept)
        plan = tsa.SparsePlan(mode=tsa.SparseMode.kDynamic, sparse_layers=[0], tau=0.0)
        out, st = tsa.sparse_attention_layer(h, plan)
        assert st.k_keep == L
    else:
        out = torch.stack([tsa.dense_causal_attention(h.q[i], h.k[0], h.v[0]) for i in range(H)])
    o = host(out)
    assert np.isfinite(o).all()
    for i in range(H):
        assert parity.rel_l2(o[i], ref) <= parity.BF16_REL_L2


def test_heavy_tailed_layer_bf16_vs_oracle(cuda, port):
    from paper_2602_03216_b200 import workloads
    L = 8192
    q, k, v = workloads.heavy_tailed_heads(8, 2, L, 128, seed=9)
    h = tsa.HeadTensors(q, k, v)
    plan = tsa.SparsePlan(mode=tsa.SparseMode.kDynamic, sparse_layers=[0], tau=0.01)
    out, st = tsa.sparse_attention_layer(h, plan)
    up = [host(t) for t in (q, k, v)]
    idx = host(st.selection.indices).astype(np.int32)
    ref = port.token_sparse_attention_sampled(up[0], up[1], up[2], idx, head_stride=3, r0=0,
                                              r1=st.k_keep, n_threads=8)
    o = host(out)
    for hh in (0, 3, 6):
        assert parity.rel_l2(o[hh], ref[hh]) <= parity.BF16_REL_L2


@pytest.mark.parametrize("dtype,L", [(torch.bfloat16, 3000), (torch.float32, 1500)])
def test_sharded_step_world1_matches_layer_bitwise(cuda, dtype, L):
    """dist.ShardedSparseAttention (stage entry points: fused K/V gather +
    zero-fill, indexed attend) equals tsa_sparse_attention_layer bit for bit,
    and rows the selection dropped are +0."""
    from paper_2602_03216_b200 import workloads
    from paper_2602_03216_b200.dist import ShardedSparseAttention
    q, k, v = workloads.heavy_tailed_heads(8, 2, L, 128, seed=4)
    q, k, v = (t.to(dtype) for t in (q, k, v))
    plan = tsa.SparsePlan(mode=tsa.SparseMode.kDynamic, sparse_layers=[0], tau=0.02)
    out, st = tsa.sparse_attention_layer(tsa.HeadTensors(q, k, v), plan)
    lay = ShardedSparseAttention(8, 2, L, 128, dtype, plan, device=q.device)
    o2 = lay.step(q, k, v)
    torch.cuda.synchronize()
    assert lay.k_keep == st.k_keep < L
    assert torch.equal(o2.view(torch.int16 if dtype == torch.bfloat16 else torch.int32),
                       out.view(torch.int16 if dtype == torch.bfloat16 else torch.int32))
    keep = torch.zeros(8, L, dtype=torch.bool, device=q.device)
    keep.scatter_(1, st.selection.indices.long(), True)
    assert bool((o2[~keep] == 0).all())


def test_graph_replay_matches_eager_bitwise(cuda):
    """tsa_sparse_attention_layer replays a captured CUDA graph from the
    second call on (same descriptor + buffers), and ShardedSparseAttention's
    step_graphed replays a torch graph: both equal the eager stage-by-stage
    step bit for bit, including after the inputs change in place."""
    from paper_2602_03216_b200 import _lib, workloads
    from paper_2602_03216_b200.dist import ShardedSparseAttention
    L = 2500
    q, k, v = workloads.heavy_tailed_heads(8, 2, L, 128, seed=9)
    plan = tsa.SparsePlan(mode=tsa.SparseMode.kDynamic, sparse_layers=[0], tau=0.02)
    h = tsa.HeadTensors(q, k, v)
    lay = ShardedSparseAttention(8, 2, L, 128, torch.bfloat16, plan, device=q.device)
    for seed in (9, 10):  # second round: new values in the same buffers
        if seed == 10:
            q2, k2, v2 = workloads.heavy_tailed_heads(8, 2, L, 128, seed=seed, sigma=2.0)
            q.copy_(q2), k.copy_(k2), v.copy_(v2)
        eager = lay.step(q, k, v).clone()
        out = torch.empty_like(q)
        n0 = _lib.load().tsa_kernel_launches()
        for _ in range(3):
            tsa.sparse_attention_layer(h, plan, out=out, stat=False)
            torch.cuda.synchronize()
            assert torch.equal(out.view(torch.int16), eager.view(torch.int16))
        assert _lib.load().tsa_kernel_launches() - n0 >= 3 * 5  # replays are counted
        g = lay.step_graphed(q, k, v).clone()
        g = lay.step_graphed(q, k, v).clone()
        assert torch.equal(g.view(torch.int16), eager.view(torch.int16))
        assert lay.graph_kernels >= 5


@pytest.mark.parametrize("dtype,L", [(torch.bfloat16, 3000), (torch.float32, 700)])
def test_host_api_equals_device_layer_bitwise(cuda, dtype, L):
    """tsa_sparse_attention_layer_host (pipelined copies, attention per head
    group) returns exactly the device-resident layer's output and budget."""
    from paper_2602_03216_b200 import workloads
    q, k, v = workloads.heavy_tailed_heads(8, 2, L, 128, seed=12)
    q, k, v = (t.to(dtype) for t in (q, k, v))
    plan = tsa.SparsePlan(mode=tsa.SparseMode.kDynamic, sparse_layers=[0], tau=0.02)
    ref, st = tsa.sparse_attention_layer(tsa.HeadTensors(q, k, v), plan)
    hq, hk, hv = (t.cpu().pin_memory() for t in (q, k, v))
    hout = torch.full(q.shape, 7.0, dtype=dtype).pin_memory()
    for groups in (0, 1, 2):
        kk = tsa.sparse_attention_layer_host(hq, hk, hv, hout, plan, n_groups=groups)
        torch.cuda.synchronize()
        assert int(kk.item()) == st.k_keep
        assert torch.equal(hout.view(torch.int16 if dtype == torch.bfloat16 else torch.int32),
                           ref.cpu().view(torch.int16 if dtype == torch.bfloat16 else torch.int32))


def test_host_api_back_to_back_calls_overlap_correctly(cuda):
    """Consecutive host-API calls without a sync alternate staging sets on two
    streams (a call's copies and scoring overlap the previous call's attention):
    three calls on different inputs into different outputs, one sync, each
    output and budget equal to its own device-resident layer."""
    from paper_2602_03216_b200 import workloads
    plan = tsa.SparsePlan(mode=tsa.SparseMode.kDynamic, sparse_layers=[0], tau=0.02)
    cases = []
    for seed in (31, 32, 33):
        q, k, v = workloads.heavy_tailed_heads(8, 2, 2500, 128, seed=seed)
        ref, st = tsa.sparse_attention_layer(tsa.HeadTensors(q, k, v), plan)
        hq, hk, hv = (t.cpu().pin_memory() for t in (q, k, v))
        hout = torch.full(q.shape, 7.0, dtype=q.dtype).pin_memory()
        cases.append((hq, hk, hv, hout, ref.cpu(), st.k_keep))
    torch.cuda.synchronize()
    kks = []
    for hq, hk, hv, hout, _, _ in cases:
        # (the clone is ordered on the caller's stream after the call's work)
        kks.append(tsa.sparse_attention_layer_host(hq, hk, hv, hout, plan).clone())
    torch.cuda.synchronize()
    for (hq, hk, hv, hout, ref, k_ref), kk in zip(cases, kks):
        assert int(kk.item()) == k_ref
        assert torch.equal(hout.view(torch.int16), ref.view(torch.int16))


def _full_size_check(port, q, k, v, tau, rows=256, head_stride=16, plan=None):
    """Default (exact) scoring at full size: scores bit-identical to the oracle,
    k_keep equal to the reference's, every index set identical, sampled
    compressed rows (the last `rows`, the costliest of the causal range) within
    the bf16 gate against the oracle on that selection, dropped rows +0."""
    from oracle.oracle import n_threads_default
    H, L = q.shape[0], q.shape[1]
    plan = plan or tsa.SparsePlan(mode=tsa.SparseMode.kDynamic, sparse_layers=[0], tau=tau)
    h = tsa.HeadTensors(q, k, v)
    out, st = tsa.sparse_attention_layer(h, plan)
    T = n_threads_default()
    up_q, up_k = host(q), host(k)
    s_ora = port.score_tokens(up_q, up_k, 64, 7, n_threads=T)
    s_gpu = host(tsa.score_tokens(h, 64, 7).s)
    assert np.array_equal(bits(s_gpu), bits(s_ora))
    k_ora = port.coverage_budget(port.aggregate_scores(s_ora), tau, 1)
    assert st.k_keep == k_ora, (st.k_keep, k_ora)
    idx = host(st.selection.indices).astype(np.int32)
    ora_idx = port.select_tokens(s_ora, k_ora, [L - 1], n_threads=T)
    assert np.array_equal(idx, ora_idx)
    keep = torch.zeros((H, L), dtype=torch.bool, device=q.device)
    keep.scatter_(1, st.selection.indices.long(), True)
    assert bool((out[~keep] == 0).all())
    kk = st.k_keep
    r0 = max(0, kk - rows)
    ref = port.token_sparse_attention_sampled(up_q, up_k, host(v), idx, head_stride=head_stride,
                                              r0=r0, r1=kk, n_threads=T)
    o = host(out)
    for hh in range(0, H, head_stride):
        sel_rows = idx[hh, r0:kk]
        assert parity.rel_l2(o[hh][sel_rows], ref[hh][sel_rows]) <= parity.BF16_REL_L2
    return out, st, s_ora, k_ora


def test_cfg3_full_size_layer(cuda, port):
    """BASELINE configs[2] at full size (L = 131072, 32 / 8 heads, bf16,
    heavy-tailed inputs, tau = 0.01) with the default (exact) scoring: scores,
    k_keep and every index set identical to the reference's (no tolerance), the
    output within the bf16 gate; tau = 0 sparse == dense bitwise at this size."""
    from paper_2602_03216_b200 import workloads
    L, H, Hkv = 131072, 32, 8
    q, k, v = workloads.heavy_tailed_heads(H, Hkv, L, 128, seed=2602)
    _full_size_check(port, q, k, v, 0.01)
    plan0 = tsa.SparsePlan(mode=tsa.SparseMode.kDynamic, sparse_layers=[0], tau=0.0)
    a, st0 = tsa.sparse_attention_layer(tsa.HeadTensors(q, k, v), plan0)
    assert st0.k_keep == L
    b, _ = tsa.sparse_attention_layer(tsa.HeadTensors(q, k, v), tsa.SparsePlan())
    assert torch.equal(a.view(torch.int16), b.view(torch.int16))


def test_cfg3_fast_scoring_at_reference_budget(cuda, port):
    """FAST scoring (opt-in) on the cfg3 layer: its budget within the FAST rule
    of the reference's, and its selection at the REFERENCE's k_keep differs only
    at tokens whose oracle score is within FAST_SCORE_REL of the head's
    threshold (the approximation's measured relative error bound)."""
    from oracle.oracle import n_threads_default
    from paper_2602_03216_b200 import workloads
    L, H, Hkv = 131072, 32, 8
    q, k, v = workloads.heavy_tailed_heads(H, Hkv, L, 128, seed=2602)
    T = n_threads_default()
    s_ora = port.score_tokens(host(q), host(k), 64, 7, n_threads=T)
    k_ora = port.coverage_budget(port.aggregate_scores(s_ora), 0.01, 1)
    plan = tsa.SparsePlan(mode=tsa.SparseMode.kDynamic, sparse_layers=[0], tau=0.01)
    _, st = tsa.sparse_attention_layer(tsa.HeadTensors(q, k, v), plan, scoring=2)
    assert abs(st.k_keep - k_ora) <= parity.FAST_BUDGET_REL * L, (st.k_keep, k_ora)
    s_fast = tsa.score_tokens(tsa.HeadTensors(q, k, v), 64, 7, scoring=2).s
    sel = host(tsa.select_tokens(tsa.HeadScores(s_fast), k_ora, [L - 1]).indices).astype(np.int32)
    ora_idx = port.select_tokens(s_ora, k_ora, [L - 1], n_threads=T)
    diffs = parity.check_index_sets(sel, ora_idx, s_ora, [L - 1], rel_tol=parity.FAST_SCORE_REL)
    assert len(diffs) <= 1e-3 * H * k_ora, len(diffs)


@pytest.mark.parametrize("tau", [0.25, 0.5, 0.75])
def test_cfg2_full_size_uniform(cuda, port, tau):
    """BASELINE configs[1] at full size: L = 32768, 32 / 8 heads, bf16, the
    reference's uniform[-1, 1) generator family (random.hpp:36-44) -- where the
    scores cluster and approximate scoring would flip many tokens -- with the
    default (exact) scoring: scores, k_keep and index sets identical to the
    reference's, outputs within the bf16 gate (bench.cpp:27 family)."""
    from paper_2602_03216_b200 import workloads
    q, k, v = workloads.uniform_heads(32, 8, 32768, 128, seed=int(tau * 100))
    out, st, _, k_ora = _full_size_check(port, q, k, v, tau, head_stride=8)
    assert abs(k_ora / 32768 - (1 - tau)) < 0.05  # k/L ~ 1 - tau on U


def test_cfg5_full_size_llama70b(cuda, port):
    """BASELINE configs[4] head geometry at full size: H = 64 / 8 (8 query heads
    per KV head: two 256-row tiles per KV group in the exact scorer), L =
    131072, bf16, heavy-tailed inputs, tau = 0.01: exact scores, k_keep and
    index sets; sampled outputs within the bf16 gate."""
    from paper_2602_03216_b200 import workloads
    q, k, v = workloads.heavy_tailed_heads(64, 8, 131072, 128, seed=70)
    _full_size_check(port, q, k, v, 0.01, head_stride=32)


@pytest.mark.parametrize("L", [1500, 4096])
def test_llama70b_gqa8_layer_vs_oracle(cuda, port, L):
    """cfg5 head geometry (8 query heads per KV head): a KV group spans two
    row tiles of the exact scorer; budget, selection and output against the
    oracle on the same bf16 inputs (exact: no tolerance)."""
    from paper_2602_03216_b200 import workloads
    H, Hkv = 16, 2
    q, k, v = workloads.heavy_tailed_heads(H, Hkv, L, 128, seed=70)
    plan = tsa.SparsePlan(mode=tsa.SparseMode.kDynamic, sparse_layers=[0], tau=0.01)
    out, st = tsa.sparse_attention_layer(tsa.HeadTensors(q, k, v), plan)
    up = [host(t) for t in (q, k, v)]
    s_ora = port.score_tokens(up[0], up[1], 64, 7, n_threads=8)
    k_ora = port.coverage_budget(port.aggregate_scores(s_ora), 0.01, 1)
    assert st.k_keep == k_ora
    idx = host(st.selection.indices).astype(np.int32)
    assert np.array_equal(idx, port.select_tokens(s_ora, k_ora, [L - 1]))
    ref = port.token_sparse_attention(up[0], up[1], up[2], idx, n_threads=8)
    o = host(out)
    for hh in range(H):
        assert parity.rel_l2(o[hh], ref[hh]) <= parity.BF16_REL_L2
    assert parity.unselected_rows_zero(o, idx, L)
