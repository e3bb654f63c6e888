"""REFERENCE-order ("exact") scoring on the B200 for bf16 inputs
(score_exact.cu): the scores must be bit-identical to the reference's f32
arithmetic on the upcast inputs -- logits in p order, glibc's expf, sequential
softmax sums, r-ordered column sums, Eigen-order pool (token_coverage.cpp:16-50)
-- so k_keep and every index set equal the reference's with no tolerance."""
import ctypes as C

import numpy as np
import pytest
import torch

import paper_2602_03216_b200 as tsa
from paper_2602_03216_b200 import _lib, workloads
from oracle.oracle import RefRng, gqa_heads

pytestmark = pytest.mark.gpu

REFERENCE = 1


def host(t):
    return t.detach().float().cpu().numpy()


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def test_expf_port_matches_host_libm(cuda, port):
    """The device expf (expf_glibc.cuh) against the host libm's expf -- the
    function std::exp(float) resolves to in the reference (tensor_ops.cpp:62)
    -- on 16 M random floats of the softmax domain [-104, -0], every float in
    [-2^-10, -0] and the underflow edge."""
    rng = np.random.default_rng(0)
    u = rng.integers(0x80000000, 0xC2D00001, size=1 << 24, dtype=np.uint64).astype(np.uint32)
    dense = np.arange(0x80000000, 0xBA800001, 997, dtype=np.uint64).astype(np.uint32)
    hx = [float.fromhex(t) for t in ("-0x1.9fe368p6", "-0x1.9fe366p6", "-0x1.9fe36ap6",
                                     "-0x1.9d1d9ep6")]
    edge = np.array(hx + [-87.33654, -88.0, -103.0, -104.0, -1e-45, -0.0, 0.0, -1.0, -0.5,
                          -2.0 ** -30], np.float32)
    x = np.concatenate([u.view(np.float32), dense.view(np.float32), edge])
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty_like(xd)
    _lib.check(_lib.load().tsa_expf(C.c_void_p(xd.data_ptr()), C.c_void_p(yd.data_ptr()), x.size,
                                    C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    y = host(yd)
    ref = port.expf(x)
    bad = np.flatnonzero(bits(y) != bits(ref))
    assert bad.size == 0, [(float(x[i]), float(y[i]), float(ref[i])) for i in bad[:5]]


SHAPES = [  # H, Hkv, L, last_q, generator
    (8, 2, 4096, 64, "tail"),
    (4, 4, 1000, 64, "uniform"),
    (8, 1, 3000, 32, "tail"),     # g * lq = 256: one full row tile
    (16, 2, 1500, 64, "tail"),    # g = 8 (70B geometry): two row tiles per KV group
    (4, 2, 700, 100, "uniform"),  # lq not a multiple of 16 / 64
    (2, 1, 50, 64, "uniform"),    # L < last_q: lq clamps to L
    (2, 2, 1, 64, "uniform"),     # L = 1
    (2, 1, 130, 7, "tail"),
    (6, 3, 2049, 64, "tail"),     # L % 64 == 1
    (32, 8, 16384, 64, "tail"),
    (8, 2, 4096, 64, "sharp"),    # logits over hundreds: tiny / zero e, the slow quotients
]


@pytest.mark.parametrize("H,Hkv,L,lq,gen", SHAPES)
def test_exact_scores_bitwise_vs_oracle(cuda, port, H, Hkv, L, lq, gen):
    if gen in ("tail", "sharp"):
        q, k, v = workloads.heavy_tailed_heads(H, Hkv, L, 128, seed=L + H, last_q=lq)
        if gen == "sharp":  # cfg4-like sharp maps (a per-layer q/k gain)
            q = (q.float() * 6.0).to(torch.bfloat16)
    else:
        qn, kn, vn = gqa_heads(RefRng(L + 7 * H), H, Hkv, L, 128)
        q, k = (torch.from_numpy(a).cuda().to(torch.bfloat16) for a in (qn, kn))
        v = None
    h = tsa.HeadTensors(q, k, v if v is not None else k)
    s = host(tsa.score_tokens(h, lq, 7, scoring=REFERENCE).s)
    s_ora = port.score_tokens(host(q), host(k), lq, 7, n_threads=8)
    bad = np.flatnonzero(bits(s) != bits(s_ora))
    assert bad.size == 0, (f"{bad.size} of {s.size} scores differ; first "
                           f"{[(int(i // L), int(i % L), s.flat[i], s_ora.flat[i]) for i in bad[:4]]}")


def test_exact_scores_match_compiled_reference(cuda, ref):
    """The same against the reference's own score_tokens compiled here
    (oracle/_ref), not only the port."""
    q, k, v = workloads.heavy_tailed_heads(8, 2, 2000, 128, seed=5)
    s = host(tsa.score_tokens(tsa.HeadTensors(q, k, v), 64, 7, scoring=REFERENCE).s)
    s_ref = ref.score_tokens(host(q), host(k), 64, 7, n_threads=8)
    assert np.array_equal(bits(s), bits(s_ref))


def test_exact_scoring_deterministic_and_shard_consistent(cuda):
    """Repeated calls are bitwise identical; a head shard computes the same
    rows as the whole layer (multi-GPU rows are exchanged verbatim)."""
    q, k, v = workloads.heavy_tailed_heads(8, 2, 5000, 128, seed=8)
    h = tsa.HeadTensors(q, k, v)
    a = tsa.score_tokens(h, 64, 7, scoring=REFERENCE).s
    b = tsa.score_tokens(h, 64, 7, scoring=REFERENCE).s
    assert torch.equal(a, b)
    from paper_2602_03216_b200 import ops
    desc = ops._heads_desc(h, last_q=64, kernel=7, scoring=REFERENCE)
    desc.head_begin, desc.head_end = 4, 8
    s = torch.full_like(a, -1.0)
    ws = ops._workspace(desc, q.device)
    _lib.check(_lib.load().tsa_score(C.byref(desc), ops._ptr(q), ops._ptr(k), ops._ptr(s),
                                     ops._ptr(ws), ops._stream(q.device)))
    torch.cuda.synchronize()
    assert torch.equal(s[4:], a[4:]) and bool((s[:4] == -1.0).all())


def _layer(q, k, v, tau):
    plan = tsa.SparsePlan(mode=tsa.SparseMode.kDynamic, sparse_layers=[0], tau=tau)
    return tsa.sparse_attention_layer(tsa.HeadTensors(q, k, v), plan, scoring=REFERENCE)
