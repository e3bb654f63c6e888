"""Generates tests/golden/*.npz from the REFERENCE itself (oracle/_ref: the
reference sources under /root/reference/proj/src compiled against the Eigen
shim).  Run in the build container:  python tests/golden/make_golden.py

Each case stores the reference's outputs for inputs that are regenerated
bit-exactly from a seed (tsa::Rng / mix_seed are bit-specified,
random.hpp:12-15, bench.cpp:31-36), so the fixtures stay small.

Cases:
  equiv_*  -- run_equiv instances (bench.cpp:225-273): MHA, uniform[-1,1),
              forced {L-1}, last_q 64, kernel 7, dynamic tau
  gqa_*    -- GQA heads (test_attention.cpp:53-61 generator), recent-window
              forced set, assorted last_q / kernel
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle.oracle import Oracle, RefRng, equiv_heads, gqa_heads  # noqa: E402

OUT = Path(__file__).resolve().parent

# run_equiv grid (bench.cpp:226-241) in its own enumeration order
GRID = [(L, H, d, tau) for L in (16, 64, 256) for H in (1, 4, 8) for d in (8, 16, 32)
        for tau in (0.0, 0.005, 0.1, 0.5, 0.99)]
EQUIV_SEED = 42
EQUIV_TRIALS = [0, 7, 33, 52, 61, 64, 88, 94, 111, 119, 127, 134]

GQA_CASES = [
    # seed, H, Hkv, L, d, last_q, kernel, tau, forced policy (0 final, 1 recent)
    (101, 8, 2, 300, 32, 64, 7, 0.05, 0),
    (102, 4, 1, 200, 16, 32, 5, 0.3, 1),
    (103, 8, 4, 129, 8, 500, 1, 0.5, 0),
    (104, 4, 4, 64, 32, 16, 3, 0.99, 1),
]


def forced_for(policy, L, last_q):
    return [L - 1] if policy == 0 else list(range(max(0, L - last_q), L))


def main():
    ref = Oracle("reference")
    cases = {}
    for trial in EQUIV_TRIALS:
        L, H, d, tau = GRID[trial % len(GRID)]
        q, k, v = equiv_heads(EQUIV_SEED, trial, L, H, d)
        s = ref.score_tokens(q, k, 64, 7)
        k_keep = ref.coverage_budget(ref.aggregate_scores(s), tau, 1)
        idx = ref.select_tokens(s, k_keep, [L - 1])
        out = ref.token_sparse_attention(q, k, v, idx, [L - 1])
        cases[f"equiv_{trial}"] = dict(
            meta=np.array([EQUIV_SEED, trial, L, H, H, d, 64, 7, 0], np.int64),
            tau=np.array(tau), scores=s, k_keep=np.array(k_keep), idx=idx, out=out)
    for (seed, H, Hkv, L, d, lq, ker, tau, pol) in GQA_CASES:
        q, k, v = gqa_heads(RefRng(seed), H, Hkv, L, d)
        s = ref.score_tokens(q, k, lq, ker)
        f = forced_for(pol, L, lq)
        k_keep = ref.coverage_budget(ref.aggregate_scores(s), tau, max(1, len(f)))
        idx = ref.select_tokens(s, k_keep, f)
        out = ref.token_sparse_attention(q, k, v, idx, f)
        cases[f"gqa_{seed}"] = dict(
            meta=np.array([seed, -1, L, H, Hkv, d, lq, ker, pol], np.int64),
            tau=np.array(tau), scores=s, k_keep=np.array(k_keep), idx=idx, out=out)
    flat = {f"{name}/{key}": val for name, c in cases.items() for key, val in c.items()}
    np.savez_compressed(OUT / "reference_cases.npz", **flat)
    print(f"wrote {len(cases)} cases to {OUT / 'reference_cases.npz'}")


def load_cases():
    """{name: dict(meta, tau, scores, k_keep, idx, out, q, k, v, forced)}"""
    z = np.load(OUT / "reference_cases.npz")
    cases = {}
    for key in z.files:
        name, field = key.split("/")
        cases.setdefault(name, {})[field] = z[key]
    for name, c in cases.items():
        seed, trial, L, H, Hkv, d, lq, ker, pol = (int(x) for x in c["meta"])
        if trial >= 0:
            c["q"], c["k"], c["v"] = equiv_heads(seed, trial, L, H, d)
        else:
            c["q"], c["k"], c["v"] = gqa_heads(RefRng(seed), H, Hkv, L, d)
        c.update(L=L, H=H, Hkv=Hkv, d=d, last_q=lq, kernel=ker, policy=pol,
                 forced=forced_for(pol, L, lq), tau=float(c["tau"]), k_keep=int(c["k_keep"]))
    return cases


if __name__ == "__main__":
    main()
