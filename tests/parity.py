"""Parity rules between the CUDA path and the CPU oracle.

* index sets: identical, except a head may differ at tokens whose oracle
  score lies within NEAR_TIE_ULPS (4) ulp of that head's selection threshold
  (the smallest kept non-forced oracle score) -- with the default (exact)
  scoring the GPU scores are bit-identical, so the sets are identical;
* k_keep: identical, except when the oracle's double prefix at the budget
  boundary lies within L * 2^-53 of tau (the double accumulation's error
  bound over L terms; the GPU sums exact 2^-62 fixed-point masses);
* FAST scoring (opt-in): scores within FAST_SCORE_REL relative, k_keep within
  FAST_BUDGET_REL * L, index sets at the reference's k_keep identical except
  tokens within FAST_SCORE_REL of the threshold (the approximation's measured
  error bound, not an fp32 near tie);
* outputs: f32 max |d| <= 1e-5 (bench.cpp:27); bf16 rel_l2 <= 1e-2
  (bench.cpp:199-214) on the oracle run with the same index sets, and
  unselected rows bitwise +0.0.
"""
from __future__ import annotations

import numpy as np

NEAR_TIE_ULPS = 4
# FAST (tensor-core) scoring: bf16 products are exact, but f32 accumulation
# order, ex2.approx and the tile-wise softmax normalisation move scores by up
# to ~1e-5 relative; near ties are judged at this relative width instead.
FAST_SCORE_REL = 2e-4
FAST_BUDGET_REL = 1e-3
F32_GATE = 1e-5
BF16_REL_L2 = 1e-2


def ulp(x):
    x = np.abs(np.asarray(x, np.float32))
    return np.spacing(x).astype(np.float64)


def check_index_sets(gpu_idx, ora_idx, ora_scores, forced, rel_tol=None):
    """Returns the list of (head, token) differences; asserts each is a near tie
    (within NEAR_TIE_ULPS ulp of the threshold, or rel_tol * threshold)."""
    diffs = []
    forced = set(int(f) for f in forced)
    for h in range(ora_idx.shape[0]):
        a, b = set(gpu_idx[h].tolist()), set(ora_idx[h].tolist())
        if a == b:
            continue
        kept = [t for t in b if t not in forced]
        thr = min(float(ora_scores[h, t]) for t in kept) if kept else 0.0
        tol = NEAR_TIE_ULPS * ulp(thr) if rel_tol is None else max(NEAR_TIE_ULPS * ulp(thr),
                                                                     rel_tol * abs(thr))
        for t in sorted(a ^ b):
            gap = abs(float(ora_scores[h, t]) - thr)
            assert gap <= tol, (f"head {h} token {t}: score {ora_scores[h, t]!r} is "
                                f"{gap:.3e} from threshold {thr!r} (> {tol:.3e})")
            diffs.append((h, t))
    return diffs


def check_budget(k_gpu, k_ora, prefix_prev, prefix_at, tau, L=None):
    if k_gpu == k_ora:
        return True
    n = L if L is not None else 1 << 20
    near = min(abs(prefix_at - tau), abs(tau - prefix_prev)) <= n * 2.0 ** -53
    assert near and abs(k_gpu - k_ora) <= 2, (
        f"k_keep {k_gpu} vs oracle {k_ora}; boundary prefix {prefix_prev!r}..{prefix_at!r}, "
        f"tau {tau}")
    return False


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    den = float(np.sum(b * b))
    num = float(np.sum((a - b) ** 2))
    return float(np.sqrt(num)) if den == 0.0 else float(np.sqrt(num / den))


def unselected_rows_zero(out, idx, L):
    """Rows off the selection are +0.0 bitwise (test_attention.cpp:275-291)."""
    out = np.ascontiguousarray(out, np.float32)
    for h in range(out.shape[0]):
        mask = np.ones(L, bool)
        mask[idx[h]] = False
        if np.any(out[h][mask].view(np.uint32) != 0):
            return False
    return True
