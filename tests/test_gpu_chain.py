"""The reference's sequential f32 total (token_coverage.cpp:58-61) on the GPU:
select.cu computes it with the chunk-monoid method (exact_chain_sum), which
must equal the one-by-one f32 chain bit for bit on every input -- exact ties
at half an ulp, binade crossings, zeros, denormals, huge dynamic range.  The
total reaches the caller through aggregate_scores: s_l = headsum / total."""
import numpy as np
import pytest
import torch

import paper_2602_03216_b200 as tsa

pytestmark = pytest.mark.gpu


def seq_total(x):
    acc = np.float32(0.0)
    for v in x.astype(np.float32):
        acc = np.float32(acc + v)
    return acc


def check(x):
    """One head: headsum == x exactly, so s_l = x / total_chain."""
    x = np.ascontiguousarray(x, np.float32)
    sl = tsa.aggregate_scores(tsa.HeadScores(torch.from_numpy(x[None]).cuda()))
    got = sl.s.cpu().numpy()
    ref = (x / seq_total(x)).astype(np.float32)
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))


def test_chain_total_vs_numpy_fast_path(cuda, port):
    """The oracle's aggregate (pinned to the reference) on a production-size row."""
    rng = np.random.default_rng(1)
    x = rng.random((4, 131072), dtype=np.float32)
    sl = tsa.aggregate_scores(tsa.HeadScores(torch.from_numpy(x).cuda()))
    assert np.array_equal(sl.s.cpu().numpy().view(np.uint32),
                          port.aggregate_scores(x).view(np.uint32))


@pytest.mark.parametrize("L", [1, 2, 7, 513, 4096, 150001])
def test_chain_uniform(cuda, L):
    check(np.random.default_rng(L).random(L, dtype=np.float32))


def test_chain_half_ulp_ties(cuda):
    """1.0 followed by exact half-ulp (2^-24) and 1.5-ulp increments: every
    addition is a tie that rounds to even -- the parity-dependent case."""
    rng = np.random.default_rng(2)
    k = rng.integers(0, 4, 100000)
    x = (k * 2.0 ** -24).astype(np.float32)
    x[0] = 1.0
    x[50000] = 3.0
    check(x)


def test_chain_ties_at_every_binade(cuda):
    """Multiples of a small power of two with a growing sum: ties recur in every
    binade the sum crosses."""
    rng = np.random.default_rng(3)
    x = (rng.integers(1, 64, 200000) * 2.0 ** -20).astype(np.float32)
    check(x)


def test_chain_heavy_tailed_zeros_denormals(cuda):
    rng = np.random.default_rng(4)
    x = np.exp(rng.normal(0.0, 6.0, 131072)).astype(np.float32)
    x[rng.integers(0, 131072, 5000)] = 0.0
    x[rng.integers(0, 131072, 5000)] = np.float32(1e-41)  # denormal
    check(x)


def test_chain_ramp_many_crossings(cuda):
    """Tiny values first, then growing: the sum crosses ~60 powers of two."""
    x = np.logspace(-30, 3, 131072).astype(np.float32)
    check(x)
    check(x[::-1].copy())


def test_chain_single_large_then_small(cuda):
    x = np.full(131072, 1e-9, np.float32)
    x[0] = 1e4
    check(x)
    x2 = np.full(131072, 1e-3, np.float32)
    x2[-1] = 1e8
    check(x2)
