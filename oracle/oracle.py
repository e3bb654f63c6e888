"""ctypes front end for the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Two implementations of the reference path live behind the same Python API:

* ``Oracle("port")``      -> ``oracle/libtsa_oracle.so``, the plain-C restatement
                             (``oracle/tsa_oracle.c``), always buildable;
* ``Oracle("reference")`` -> ``oracle/_ref/libtsa_ref.so``, the reference's own
                             sources compiled against the Eigen shim
                             (``oracle/Makefile`` target ``ref``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs import this module.  The product path
(``paper_2602_03216_b200``) never does.

Arrays are numpy, C-contiguous: q ``[H, L, d]`` f32, k/v ``[Hkv, L, d]`` f32,
scores ``[H, L]`` f32, index lists ``[H, k_keep]`` int32 (reference layout,
attention.hpp:16-25, selection.hpp:12-21).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
PORT_SO = HERE / "libtsa_oracle.so"
REF_SO = HERE / "_ref" / "libtsa_ref.so"

_f32p = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_I = C.c_int
_D = C.c_double


class OracleError(ValueError):
    """Precondition failure reported by the oracle (reference: std::invalid_argument)."""


def build(ref: bool = False) -> None:
    """Compile the restatement (and, with ``ref``, the reference) via oracle/Makefile."""
    targets = ["all"] + (["ref"] if ref else [])
    subprocess.run(["make", "-s", "-C", str(HERE), *targets], check=True)


def n_threads_default() -> int:
    return max(1, len(os.sched_getaffinity(0)))


class Oracle:
    def __init__(self, kind: str = "port"):
        self.kind = kind
        path = PORT_SO if kind == "port" else REF_SO
        if not path.exists():
            build(ref=(kind == "reference"))
        self.lib = C.CDLL(str(path))
        self._bind()

    # ------------------------------------------------------------ binding
    def _bind(self):
        L = self.lib
        if self.kind == "port":
            p = "tsa_oracle_"
            L.tsa_oracle_last_error.restype = C.c_char_p
            L.tsa_oracle_score_tokens.argtypes = [_f32p, _f32p, _I, _I, _I, _I, _I, _I, _f32p, _I]
            L.tsa_oracle_aggregate_scores.argtypes = [_f32p, _I, _I, _f32p]
            L.tsa_oracle_coverage_budget_ex.argtypes = [_f32p, _I, _D, _I, C.POINTER(_I),
                                                        C.POINTER(_D), C.POINTER(_D)]
            L.tsa_oracle_fixed_budget.argtypes = [_I, _D, _I, C.POINTER(_I)]
            L.tsa_oracle_select_tokens.argtypes = [_f32p, _I, _I, _I, _i32p, _I, _i32p, _I]
            L.tsa_oracle_dense_causal_attention.argtypes = [_f32p, _f32p, _f32p, _I, _I, _f32p]
            L.tsa_oracle_masked_sparse_oracle.argtypes = [_f32p, _f32p, _f32p, _I, _I, _i32p, _I,
                                                          _f32p]
            L.tsa_oracle_token_sparse_attention.argtypes = [_f32p, _f32p, _f32p, _I, _I, _I, _I,
                                                            _i32p, _I, _f32p, _I]
            L.tsa_oracle_token_sparse_attention_sampled.argtypes = [
                _f32p, _f32p, _f32p, _I, _I, _I, _I, _i32p, _I, _I, _I, _I, _f32p, _I]
            L.tsa_oracle_avg_pool_1d.argtypes = [_f32p, _I, _I, _f32p]
            L.tsa_oracle_rms_norm.argtypes = [_f32p, _f32p, _I, _I, C.c_float, _f32p]
            L.tsa_oracle_apply_rope.argtypes = [_f32p, _I, _I, C.c_float, _f32p]
            L.tsa_oracle_project_qkv.argtypes = [_f32p, _f32p, _f32p, _f32p, _I, _I, _I, _I, _I,
                                                 C.c_float, _f32p, _f32p, _f32p]
            L.tsa_oracle_compute_drift.argtypes = [_f32p, _I, _I, _I, _D, _f64p]
            L.tsa_oracle_select_sparse_layers.argtypes = [_f64p, _I, _D, _f64p, _i32p, C.POINTER(_I)]
            L.tsa_oracle_rng_new.restype = C.c_void_p
            L.tsa_oracle_expf.argtypes = [_f32p, _f32p, C.c_int64]
            L.tsa_oracle_expf.restype = None
            L.tsa_oracle_rng_new.argtypes = [C.c_uint64]
            L.tsa_oracle_rng_free.argtypes = [C.c_void_p]
            L.tsa_oracle_rng_fill.argtypes = [C.c_void_p, C.c_int64, C.c_float, _f32p]
            L.tsa_oracle_rng_raw.restype = C.c_uint64
            L.tsa_oracle_rng_raw.argtypes = [C.c_void_p]
            L.tsa_oracle_mix_seed.restype = C.c_uint64
            L.tsa_oracle_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        else:
            L.tsa_ref_last_error.restype = C.c_char_p
            L.tsa_ref_score_tokens.argtypes = [_f32p, _f32p, _I, _I, _I, _I, _I, _I, _f32p]
            L.tsa_ref_score_tokens_mt.argtypes = [_f32p, _f32p, _I, _I, _I, _I, _I, _I, _f32p, _I]
            L.tsa_ref_aggregate_scores.argtypes = [_f32p, _I, _I, _f32p]
            L.tsa_ref_coverage_budget.argtypes = [_f32p, _I, _D, _I, C.POINTER(_I)]
            L.tsa_ref_fixed_budget.argtypes = [_I, _D, _I, C.POINTER(_I)]
            L.tsa_ref_select_tokens.argtypes = [_f32p, _I, _I, _I, _i32p, _I, _i32p]
            L.tsa_ref_dense_causal_attention.argtypes = [_f32p, _f32p, _f32p, _I, _I, _f32p]
            L.tsa_ref_masked_sparse_oracle.argtypes = [_f32p, _f32p, _f32p, _I, _I, _i32p, _I,
                                                       _f32p]
            L.tsa_ref_token_sparse_attention.argtypes = [_f32p, _f32p, _f32p, _I, _I, _I, _I,
                                                         _i32p, _I, _i32p, _I, _f32p]
            L.tsa_ref_tsa_head_prefix.argtypes = [_f32p, _f32p, _f32p, _I, _I, _I, _I, _i32p, _I,
                                                  _I, _I, _f32p]
            L.tsa_ref_rms_norm.argtypes = [_f32p, _f32p, _I, _I, C.c_float, _f32p]
            L.tsa_ref_apply_rope.argtypes = [_f32p, _I, _I, C.c_float, _f32p]
            L.tsa_ref_project_qkv.argtypes = [_f32p, _f32p, _f32p, _f32p, _I, _I, _I, _I, _I,
                                              C.c_float, _f32p, _f32p, _f32p]
            L.tsa_ref_compute_drift.argtypes = [_f32p, _I, _I, _I, _D, _f64p]
            L.tsa_ref_estimate_flops.argtypes = [_I, _I, _I, _i32p, _I, _I, _I, _f64p]
            L.tsa_ref_select_sparse_layers.argtypes = [_f64p, _I, _D, _f64p, _i32p, C.POINTER(_I)]

    def _check(self, rc: int):
        if rc != 0:
            fn = self.lib.tsa_oracle_last_error if self.kind == "port" else self.lib.tsa_ref_last_error
            raise OracleError(fn().decode())

    # ---------------------------------------------------------------- API
    def score_tokens(self, q, k, last_q=64, kernel=7, n_threads=None):
        """token_coverage.cpp:16-50 -> s [H, L] f32."""
        q, k = _f32(q), _f32(k)
        H, L, d = q.shape
        Hkv = k.shape[0]
        s = np.empty((H, L), np.float32)
        if self.kind == "port":
            self._check(self.lib.tsa_oracle_score_tokens(q, k, H, Hkv, L, d, last_q, kernel, s,
                                                         n_threads or 1))
        elif n_threads and n_threads > 1:
            self._check(self.lib.tsa_ref_score_tokens_mt(q, k, H, Hkv, L, d, last_q, kernel, s,
                                                         n_threads))
        else:
            self._check(self.lib.tsa_ref_score_tokens(q, k, H, Hkv, L, d, last_q, kernel, s))
        return s

    def expf(self, x):
        """The host libm's expf, elementwise (std::exp(float), tensor_ops.cpp:62)."""
        x = _f32(x)
        y = np.empty_like(x)
        self.lib.tsa_oracle_expf(x.ravel(), y.ravel(), x.size) if self.kind == "port" else None
        return y

    def aggregate_scores(self, s):
        """token_coverage.cpp:52-66 -> s_l [L] f32."""
        s = _f32(s)
        H, L = s.shape
        out = np.empty(L, np.float32)
        fn = (self.lib.tsa_oracle_aggregate_scores if self.kind == "port"
              else self.lib.tsa_ref_aggregate_scores)
        self._check(fn(s, H, L, out))
        return out

    def coverage_budget(self, sl, tau, min_keep=1, with_prefix=False):
        """token_coverage.cpp:68-96 -> k_keep (and the double prefix before/at the crossing)."""
        sl = _f32(sl)
        k = _I()
        if self.kind == "port":
            pp, pa = _D(), _D()
            self._check(self.lib.tsa_oracle_coverage_budget_ex(sl, sl.size, tau, min_keep,
                                                               C.byref(k), C.byref(pp), C.byref(pa)))
            return (k.value, pp.value, pa.value) if with_prefix else k.value
        self._check(self.lib.tsa_ref_coverage_budget(sl, sl.size, tau, min_keep, C.byref(k)))
        return k.value

    def fixed_budget(self, L, s, min_keep=1):
        k = _I()
        fn = self.lib.tsa_oracle_fixed_budget if self.kind == "port" else self.lib.tsa_ref_fixed_budget
        self._check(fn(L, s, min_keep, C.byref(k)))
        return k.value

    def select_tokens(self, s, k_keep, forced=(), n_threads=None):
        """token_coverage.cpp:111-152 -> idx [H, k_keep] int32 ascending."""
        s = _f32(s)
        H, L = s.shape
        f = np.ascontiguousarray(np.asarray(forced, np.int32).reshape(-1))
        out = np.empty((H, max(k_keep, 0)), np.int32)
        if self.kind == "port":
            self._check(self.lib.tsa_oracle_select_tokens(s, H, L, k_keep, f, f.size, out,
                                                          n_threads or 1))
        else:
            self._check(self.lib.tsa_ref_select_tokens(s, H, L, k_keep, f, f.size, out))
        return out

    def dense_causal_attention(self, q, k, v):
        q, k, v = _f32(q), _f32(k), _f32(v)
        n, d = q.shape
        out = np.empty((n, d), np.float32)
        fn = (self.lib.tsa_oracle_dense_causal_attention if self.kind == "port"
              else self.lib.tsa_ref_dense_causal_attention)
        self._check(fn(q, k, v, n, d, out))
        return out

    def masked_sparse_oracle(self, q, k, v, s):
        q, k, v = _f32(q), _f32(k), _f32(v)
        n, d = q.shape
        s = np.ascontiguousarray(np.asarray(s, np.int32))
        out = np.empty((n, d), np.float32)
        fn = (self.lib.tsa_oracle_masked_sparse_oracle if self.kind == "port"
              else self.lib.tsa_ref_masked_sparse_oracle)
        self._check(fn(q, k, v, n, d, s, s.size, out))
        return out

    def token_sparse_attention(self, q, k, v, idx, forced=(), n_threads=None):
        """attention.cpp:74-99 -> out [H, L, d] f32."""
        q, k, v = _f32(q), _f32(k), _f32(v)
        H, L, d = q.shape
        idx = np.ascontiguousarray(idx, np.int32)
        out = np.empty((H, L, d), np.float32)
        if self.kind == "port":
            self._check(self.lib.tsa_oracle_token_sparse_attention(
                q, k, v, H, k.shape[0], L, d, idx, idx.shape[1], out, n_threads or 1))
        else:
            f = np.ascontiguousarray(np.asarray(forced, np.int32).reshape(-1))
            self._check(self.lib.tsa_ref_token_sparse_attention(
                q, k, v, H, k.shape[0], L, d, idx, idx.shape[1], f, f.size, out))
        return out

    def token_sparse_attention_sampled(self, q, k, v, idx, head_stride, r0, r1, n_threads=None):
        """Rows [r0, r1) of the compressed output of heads 0, stride, 2*stride, ...
        scattered into [H, L, d] (other rows/heads zero).  Port only."""
        assert self.kind == "port"
        q, k, v = _f32(q), _f32(k), _f32(v)
        H, L, d = q.shape
        idx = np.ascontiguousarray(idx, np.int32)
        out = np.zeros((H, L, d), np.float32)
        self._check(self.lib.tsa_oracle_token_sparse_attention_sampled(
            q, k, v, H, k.shape[0], L, d, idx, idx.shape[1], head_stride, r0, r1, out,
            n_threads or 1))
        return out

    def tsa_head_prefix(self, q, k, v, idx, h, m):
        """Reference only: first m compressed output rows of head h (bench sample)."""
        assert self.kind == "reference"
        q, k, v = _f32(q), _f32(k), _f32(v)
        H, L, d = q.shape
        idx = np.ascontiguousarray(idx, np.int32)
        out = np.empty((m, d), np.float32)
        self._check(self.lib.tsa_ref_tsa_head_prefix(q, k, v, H, k.shape[0], L, d, idx,
                                                     idx.shape[1], h, m, out))
        return out

    # ------------------------------------------- attention-branch producer
    def _fn(self, name):
        return getattr(self.lib, ("tsa_oracle_" if self.kind == "port" else "tsa_ref_") + name)

    def rms_norm(self, x, gain, eps):
        """model.cpp:81-94 -> [rows, cols] f32."""
        x, gain = _f32(x), _f32(gain)
        out = np.empty_like(x)
        self._check(self._fn("rms_norm")(x, gain, x.shape[0], x.shape[1], eps, out))
        return out

    def apply_rope(self, x, theta):
        """model.cpp:96-123 at positions 0..rows-1 -> [rows, cols] f32."""
        x = _f32(x)
        out = np.empty_like(x)
        self._check(self._fn("apply_rope")(x, x.shape[0], x.shape[1], theta, out))
        return out

    def project_qkv(self, x_norm, wq, wk, wv, H, Hkv, d, theta):
        """model.cpp:139-158 -> q [H, L, d], k [Hkv, L, d], v [Hkv, L, d] f32."""
        x_norm, wq, wk, wv = _f32(x_norm), _f32(wq), _f32(wk), _f32(wv)
        L, D = x_norm.shape
        q = np.empty((H, L, d), np.float32)
        k = np.empty((Hkv, L, d), np.float32)
        v = np.empty((Hkv, L, d), np.float32)
        self._check(self._fn("project_qkv")(x_norm, wq, wk, wv, L, D, H, Hkv, d, theta, q, k, v))
        return q, k, v

    def compute_drift(self, hidden, epsilon=1e-6):
        """drift.cpp:14-45: hidden [n_mats, rows, cols] -> R [n_mats - 1] (double)."""
        h = _f32(hidden)
        R = np.empty(h.shape[0] - 1, np.float64)
        self._check(self._fn("compute_drift")(h, h.shape[0], h.shape[1], h.shape[2], epsilon, R))
        return R

    def select_sparse_layers(self, R, delta):
        """drift.cpp:47-65 -> (R_hat, sparse layer list)."""
        R = np.ascontiguousarray(R, np.float64)
        R_hat = np.empty_like(R)
        layers = np.empty(R.size, np.int32)
        m = _I()
        self._check(self._fn("select_sparse_layers")(R, R.size, delta, R_hat, layers, C.byref(m)))
        return R_hat, layers[:m.value].tolist()

    def estimate_flops(self, seq_len, d_head, n_heads, k_keep, last_q=64, kernel=7):
        """flops.cpp:12-51 (reference only); k_keep entries None = dense layer."""
        assert self.kind == "reference"
        kk = np.array([-1 if k is None else k for k in k_keep], np.int32)
        out = np.empty(6, np.float64)
        self._check(self.lib.tsa_ref_estimate_flops(seq_len, d_head, n_heads, kk, kk.size, last_q,
                                                    kernel, out))
        keys = ["dense_flops", "sparse_flops", "overhead_flops", "attn_ratio", "est_speedup",
                "avg_map_sparsity"]
        return dict(zip(keys, out.tolist()))

    def avg_pool_1d(self, v, kernel):
        assert self.kind == "port"
        v = _f32(v)
        out = np.empty_like(v)
        self._check(self.lib.tsa_oracle_avg_pool_1d(v, v.size, kernel, out))
        return out


# ------------------------------------------------------------------ inputs
class RefRng:
    """tsa::Rng (random.hpp:16-33) via the port's mt19937_64."""

    _lib = None

    def __init__(self, seed: int):
        if RefRng._lib is None:
            RefRng._lib = Oracle("port").lib
        self._h = RefRng._lib.tsa_oracle_rng_new(C.c_uint64(seed & (2**64 - 1)))

    def __del__(self):
        if getattr(self, "_h", None) and RefRng._lib is not None:
            RefRng._lib.tsa_oracle_rng_free(self._h)

    def random_matrix(self, rows: int, cols: int, scale: float = 1.0) -> np.ndarray:
        out = np.empty((rows, cols), np.float32)
        RefRng._lib.tsa_oracle_rng_fill(self._h, rows * cols, scale, out)
        return out

    def raw(self) -> int:
        return RefRng._lib.tsa_oracle_rng_raw(self._h)

    def below(self, n: int) -> int:
        return int(self.raw() % n)


def mix_seed(seed: int, stream: int) -> int:
    """bench.cpp:31-36 (splitmix64 stream separation)."""
    if RefRng._lib is None:
        RefRng._lib = Oracle("port").lib
    return RefRng._lib.tsa_oracle_mix_seed(C.c_uint64(seed), C.c_uint64(stream))


def equiv_heads(seed: int, trial: int, L: int, H: int, d: int):
    """run_equiv's inputs (bench.cpp:247-253): MHA, per head q, k, v uniform[-1,1)."""
    rng = RefRng(mix_seed(seed, 1000 + trial))
    q = np.empty((H, L, d), np.float32)
    k = np.empty((H, L, d), np.float32)
    v = np.empty((H, L, d), np.float32)
    for h in range(H):
        q[h] = rng.random_matrix(L, d)
        k[h] = rng.random_matrix(L, d)
        v[h] = rng.random_matrix(L, d)
    return q, k, v


def gqa_heads(rng: RefRng, H: int, Hkv: int, L: int, d: int):
    """The reference tests' random_heads (test_attention.cpp:53-61): all q first,
    then (k, v) per KV head."""
    q = np.stack([rng.random_matrix(L, d) for _ in range(H)])
    k = np.empty((Hkv, L, d), np.float32)
    v = np.empty((Hkv, L, d), np.float32)
    for h in range(Hkv):
        k[h] = rng.random_matrix(L, d)
        v[h] = rng.random_matrix(L, d)
    return q, k, v


def rel_l2(a, b) -> float:
    """bench.cpp:199-214 (the reference's output_deviation metric), in double."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    num = float(np.sum((a - b) ** 2))
    den = float(np.sum(b ** 2))
    return float(np.sqrt(num)) if den == 0.0 else float(np.sqrt(num) / np.sqrt(den))


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)
