"""CPU model of the chain-free exact f32 sum (csrc/chain_sum.cuh): the
sequential sum S_i = RN(S_{i-1} + x_i) of non-negative floats, reproduced from
per-chunk (increment, parity) folds under a guessed binade and a walk with the
exact running sum.  Pins the arithmetic argument on adversarial inputs against
numpy's one-by-one float32 chain (the reference's total, token_coverage.cpp:58-61)."""
import numpy as np
import pytest

TWO24 = 1 << 24


def seq_sum(x):
    s = np.float32(0.0)
    for v in x:
        s = np.float32(s + v)
    return s


def binade(v):
    """E with 2^E <= v < 2^(E+1) for a normal float32 v > 0, else None."""
    b = np.float32(v).view(np.uint32)
    e = int(b >> 23) & 0xFF
    return None if e == 0 or e == 0xFF else e - 127


def fold(chunk, E):
    """(inc0, inc1, valid): the chunk's total increment in units of u = 2^(E-23)
    for a start significand of parity 0 / 1 (chain_fold_elem), or invalid if an
    element reaches 2^24 u (the chunk must cross a binade)."""
    inc = [0, 0]
    q = [0, 1]
    scale = 2.0 ** (23 - E)
    for v in chunk:
        y = float(v) * scale  # exact: power-of-two scaling of a float32
        if y >= TWO24:
            return None
        k = int(np.floor(y))
        f = y - k
        for p in (0, 1):
            if f == 0.5:
                e = k + ((q[p] + k) & 1)  # ties to even: a + k + r even
            else:
                e = k + (1 if f > 0.5 else 0)
            inc[p] += e
            q[p] = (q[p] + e) & 1
    return inc


def chain_free_sum(x, C=64):
    x = np.asarray(x, np.float32)
    chunks = [x[i:i + C] for i in range(0, len(x), C)]
    approx = np.concatenate([[0.0], np.cumsum([float(c.astype(np.float64).sum()) for c in chunks])])
    S = np.float32(0.0)
    walked = elementwise = 0
    for ci, c in enumerate(chunks):
        E_guess = binade(np.float32(approx[ci])) if approx[ci] > 0 else None
        Es = binade(S) if S > 0 else None
        if E_guess is not None and Es == E_guess:
            f = fold(c, E_guess)
            if f is not None:
                bits = int(np.float32(S).view(np.uint32))
                a = (bits & 0x7FFFFF) | 0x800000
                inc = f[a & 1]
                if a + inc <= TWO24:
                    S = np.float32((a + inc) * 2.0 ** (Es - 23))  # exact
                    walked += 1
                    continue
        for v in c:  # crossing chunk or wrong guess: element by element
            S = np.float32(S + v)
        elementwise += 1
    return S, walked, elementwise


CASES = {
    "uniform": lambda r: r.random(5000, dtype=np.float32),
    "half_ulp_ties": lambda r: np.concatenate(
        [[1.0], (r.integers(0, 4, 6000) * 2.0 ** -24)]).astype(np.float32),
    "ties_every_binade": lambda r: (r.integers(1, 64, 6000) * 2.0 ** -20).astype(np.float32),
    "heavy_tail_zeros_denormals": lambda r: np.where(
        r.random(6000) < 0.1, np.float32(1e-41),
        np.exp(r.normal(0, 6, 6000))).astype(np.float32),
    "ramp_many_crossings": lambda r: np.logspace(-30, 3, 6000).astype(np.float32),
    "ramp_down": lambda r: np.logspace(3, -30, 6000).astype(np.float32),
    "large_then_small": lambda r: np.concatenate([[1e4], np.full(6000, 1e-9)]).astype(np.float32),
}


@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("C", [8, 64, 256])
def test_chain_free_sum_equals_the_sequential_chain(name, C):
    x = CASES[name](np.random.default_rng(7))
    got, walked, _ = chain_free_sum(x, C)
    ref = seq_sum(x)
    assert np.float32(got).view(np.uint32) == ref.view(np.uint32), (name, C, got, ref)
    if name == "uniform" and C == 64:
        assert walked > len(x) // C // 2  # the fast path carries most chunks


def test_tie_rule_matters():
    """Without the parity-dependent tie rule the model would diverge: a run of
    exact half-ulp additions to an odd significand rounds up, to an even one
    stays -- the fold tracks both start parities."""
    odd = np.float32(1.0) + np.float32(2.0 ** -23)  # odd significand
    x = np.array([odd] + [2.0 ** -24] * 7, np.float32)
    assert chain_free_sum(x, 4)[0] == seq_sum(x)
    even = np.array([1.0] + [2.0 ** -24] * 7, np.float32)
    assert chain_free_sum(even, 4)[0] == seq_sum(even) == np.float32(1.0)
