"""Report / harness compatibility with the reference's ``tsa bench`` commands.

``run_sweep`` and ``run_fixed_vs_dynamic`` produce the reference's rows
(bench.cpp:275-314 -- tau, seq_len, avg_k_keep, map_sparsity, est_speedup;
mode, param, ..., output_deviation) in the reference's JSON / CSV layouts
(bench.cpp:421-477, with its "# config" / "# reference" CSV header lines and
the paper's operating points), and add the MEASURED columns next to the
reference's FLOP-model estimate: the B200 latency of the stack under the plan
(``ms``), of the same stack dense (``dense_ms``) and their ratio
(``measured_speedup``).

The model is the cfg4 attention stack (stack.py) rather than the reference's
full toy transformer: every layer is the attention branch of layer_forward, the
sparse layers are chosen by drift calibration (drift.cpp:67-80, delta), and
``output_deviation`` is the rel_l2 (bench.cpp:199-214) of the final residual
stream against the dense run (the reference compares logits).

    python -m paper_2602_03216_b200.report sweep --seq-lens 16384,65536 --taus 0.005,0.01
    python -m paper_2602_03216_b200.report fixed-vs-dynamic --seq-len 65536 --format csv
"""
from __future__ import annotations

import argparse
import json
import math
import sys
from typing import List, Optional, Sequence

import torch

from . import ops
from .ops import SparseMode, SparsePlan

REFERENCE_POINTS_SWEEP = [  # bench.cpp:159-163
    {"tau": 0.005, "seq_len": 131072, "map_sparsity_pct": 54.44},
    {"tau": 0.01, "seq_len": 131072, "map_sparsity_pct": 67.36}]
REFERENCE_POINTS_FVD = [  # bench.cpp:165-171
    {"mode": "fixed", "param": 0.3, "map_sparsity_pct": 50.96, "speedup": 1.32},
    {"mode": "fixed", "param": 0.5, "map_sparsity_pct": 74.95, "speedup": 1.57},
    {"mode": "dynamic", "param": 0.005, "map_sparsity_pct": 54.44, "speedup": 1.36},
    {"mode": "dynamic", "param": 0.01, "map_sparsity_pct": 67.36, "speedup": 1.51}]


def estimate_flops(seq_len: int, d_head: int, n_heads: int, k_keep: Sequence[Optional[int]],
                   last_q: int = 64, kernel: int = 7) -> dict:
    """flops.cpp:12-51: the reference's FLOP model (None = a dense layer)."""
    if min(seq_len, d_head, n_heads, last_q, kernel) < 1:
        raise ops.InvalidArgument("estimate_flops: dimensions must be positive")
    L, d, H = float(seq_len), float(d_head), float(n_heads)
    dense_per_layer = 4.0 * L * L * d * H
    lq = min(float(last_q), L)
    r = {"dense_flops": 0.0, "sparse_flops": 0.0, "overhead_flops": 0.0, "map_sparsity": []}
    for budget in k_keep:
        r["dense_flops"] += dense_per_layer
        if budget is None:
            r["sparse_flops"] += dense_per_layer
            continue
        if budget < 1 or budget > seq_len:
            raise ops.InvalidArgument(f"estimate_flops: k_keep {budget} outside [1, {seq_len}]")
        k = float(budget)
        r["sparse_flops"] += 4.0 * k * k * d * H
        r["overhead_flops"] += H * (2.0 * lq * L * d + L * (kernel + math.log2(L))
                                    + 6.0 * k * d + L * d)
        r["map_sparsity"].append(1.0 - (k / L) * (k / L))
    r["attn_ratio"] = r["dense_flops"] / r["sparse_flops"] if r["sparse_flops"] > 0 else 1.0
    total = r["sparse_flops"] + r["overhead_flops"]
    r["est_speedup"] = r["dense_flops"] / total if total > 0 else 1.0
    ms = r["map_sparsity"]
    r["avg_map_sparsity"] = sum(ms) / len(ms) if ms else 0.0
    return r


def rel_l2(a: torch.Tensor, b: torch.Tensor) -> float:
    """bench.cpp:199-214: |a - b|_F / |b|_F accumulated in double."""
    a64, b64 = a.double(), b.double()
    den = float((b64 * b64).sum())
    return math.sqrt(float(((a64 - b64) ** 2).sum()) / den) if den > 0 else 0.0


def _metrics(stack, L: int, last_q: int, kernel: int) -> dict:
    """bench.cpp:179-195 from the stack's per-layer budgets."""
    kk = stack.k_keep.cpu().tolist()
    budgets = [kk[i] if stack.plan.is_sparse_layer(i) else None for i in range(stack.n_layers)]
    fr = estimate_flops(L, stack.d, stack.H, budgets, last_q, kernel)
    sparse = [b for b in budgets if b is not None]
    return {"avg_k_keep": sum(sparse) / len(sparse) if sparse else float(L),
            "map_sparsity": fr["avg_map_sparsity"], "est_speedup": fr["est_speedup"]}


def _time(fn, reps: int = 2) -> float:
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


class _Harness:
    def __init__(self, args):
        self.args = args

    def stack(self, L: int):
        from .stack import PrefillAttentionStack, structured_hidden
        a = self.args
        st = PrefillAttentionStack(a.n_layers, a.n_heads, a.n_kv_heads, a.d_head, a.d_model, L,
                                   SparsePlan(), seed=a.seed, device="cuda")
        x0 = structured_hidden(L, a.d_model, seed=a.seed + 1)
        prof = st.calibrate(x0, delta=a.delta, epsilon=a.epsilon)
        return st, x0, prof

    def run(self, st, x0, plan: Optional[SparsePlan], dense: bool = False):
        if plan is not None:
            st.set_plan(plan)
        x = torch.empty_like(x0)

        def once():
            x.copy_(x0)
            st.forward(x, dense=dense)
        ms = _time(once, self.args.reps)
        return x, ms

    def plan(self, mode: SparseMode, layers: List[int], tau=0.0, s=0.0) -> SparsePlan:
        a = self.args
        return SparsePlan(mode=mode, sparse_layers=list(layers), tau=tau, s_fixed=s,
                          last_q=a.last_q, kernel=a.kernel)


def run_sweep(args) -> List[dict]:
    """bench.cpp:275-292 + measured latency."""
    h = _Harness(args)
    rows = []
    for L in args.seq_lens:
        st, x0, prof = h.stack(L)
        _, dense_ms = h.run(st, x0, None, dense=True)
        for tau in args.taus:
            _, ms = h.run(st, x0, h.plan(SparseMode.kDynamic, prof["sparse_layers"], tau=tau))
            m = _metrics(st, L, args.last_q, args.kernel)
            rows.append({"tau": tau, "seq_len": L, **m, "ms": round(ms, 3),
                         "dense_ms": round(dense_ms, 3),
                         "measured_speedup": round(dense_ms / ms, 4)})
        del st, x0
        torch.cuda.empty_cache()
    return rows


def run_fixed_vs_dynamic(args) -> List[dict]:
    """bench.cpp:294-314 + measured latency."""
    h = _Harness(args)
    L = args.seq_len
    st, x0, prof = h.stack(L)
    xd, dense_ms = h.run(st, x0, None, dense=True)
    dense_out = xd.clone()
    rows = []
    cases = [(SparseMode.kFixed, s) for s in args.s_fixed] + \
            [(SparseMode.kDynamic, t) for t in args.taus]
    for mode, p in cases:
        plan = h.plan(mode, prof["sparse_layers"], tau=p if mode == SparseMode.kDynamic else 0.0,
                      s=p if mode == SparseMode.kFixed else 0.0)
        x, ms = h.run(st, x0, plan)
        m = _metrics(st, L, args.last_q, args.kernel)
        rows.append({"mode": "fixed" if mode == SparseMode.kFixed else "dynamic", "param": p, **m,
                     "output_deviation": rel_l2(x, dense_out), "ms": round(ms, 3),
                     "dense_ms": round(dense_ms, 3), "measured_speedup": round(dense_ms / ms, 4)})
    return rows


def _config(args) -> dict:
    keys = ["command", "seed", "seq_len", "seq_lens", "taus", "delta", "epsilon", "last_q",
            "kernel", "s_fixed", "n_layers", "n_heads", "n_kv_heads", "d_head", "d_model"]
    return {k: getattr(args, k) for k in keys}


def _fmt(x) -> str:
    return f"{x:.6g}" if isinstance(x, float) else str(x)


def emit(args, rows: List[dict], out) -> None:
    sweep = args.command == "sweep"
    cols = (["tau", "seq_len", "avg_k_keep", "map_sparsity", "est_speedup"] if sweep else
            ["mode", "param", "avg_k_keep", "map_sparsity", "est_speedup", "output_deviation"])
    cols += ["ms", "dense_ms", "measured_speedup"]
    ref = REFERENCE_POINTS_SWEEP if sweep else REFERENCE_POINTS_FVD
    if args.format == "csv":
        out.write("# config " + json.dumps(_config(args)) + "\n")
        out.write("# reference " + json.dumps(ref) + "\n")
        out.write(",".join(cols) + "\n")
        for r in rows:
            out.write(",".join(_fmt(r[c]) for c in cols) + "\n")
    else:
        out.write(json.dumps({"command": args.command, "config": _config(args),
                              "reference_points": ref,
                              "rows": [{c: r[c] for c in cols} for r in rows]}, indent=2) + "\n")


def main(argv=None) -> int:
    p = argparse.ArgumentParser(prog="python -m paper_2602_03216_b200.report")
    p.add_argument("command", choices=["sweep", "fixed-vs-dynamic"])
    p.add_argument("--seq-len", type=int, default=16384)
    p.add_argument("--seq-lens", type=lambda s: [int(x) for x in s.split(",")], default=None)
    p.add_argument("--taus", type=lambda s: [float(x) for x in s.split(",")],
                   default=[0.005, 0.01])
    p.add_argument("--s-fixed", type=lambda s: [float(x) for x in s.split(",")],
                   default=[0.3, 0.5])
    p.add_argument("--delta", type=float, default=0.5)
    p.add_argument("--epsilon", type=float, default=1e-6)
    p.add_argument("--last-q", type=int, default=64)
    p.add_argument("--kernel", type=int, default=7)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--n-layers", type=int, default=8)
    p.add_argument("--n-heads", type=int, default=32)
    p.add_argument("--n-kv-heads", type=int, default=8)
    p.add_argument("--d-head", type=int, default=128)
    p.add_argument("--d-model", type=int, default=4096)
    p.add_argument("--reps", type=int, default=2)
    p.add_argument("--format", choices=["json", "csv"], default="json")
    p.add_argument("--out", type=str, default="")
    args = p.parse_args(argv)
    if args.seq_lens is None:
        args.seq_lens = [args.seq_len]
    rows = run_sweep(args) if args.command == "sweep" else run_fixed_vs_dynamic(args)
    if args.out:
        with open(args.out, "w") as f:
            emit(args, rows, f)
    else:
        emit(args, rows, sys.stdout)
    return 0


if __name__ == "__main__":
    sys.exit(main())
