"""Host-side mirror of the reference operator API over the CUDA C ABI.

Same names, argument meaning and error behaviour as
/root/reference/proj/include/tsa/{attention,token_coverage,model}.hpp, with
tensors in device memory:

==========================  ================================================
reference (C++/Eigen)        here (torch CUDA tensors, via libtsa_b200.so)
==========================  ================================================
HeadTensors{q[H],k[Hkv],v}   HeadTensors(q [H,L,d], k [Hkv,L,d], v [Hkv,L,d])
HeadScores{s[HxL]}           HeadScores(s [H,L] f32)
LayerScores{s[L]}            LayerScores(s [L] f32)
TokenSelection               TokenSelection(indices [H,k] int32, k_keep, tau, forced)
score_tokens                 score_tokens(heads, last_q, kernel)
aggregate_scores             aggregate_scores(hs)
coverage_budget              coverage_budget(sl, tau, min_keep)
fixed_budget                 fixed_budget(seq_len, s, min_keep)
select_tokens                select_tokens(hs, k_keep, forced)
dense_causal_attention       dense_causal_attention(q, k, v)
token_sparse_attention       token_sparse_attention(heads, sel, inner=None)
layer_forward sparse branch  sparse_attention_layer(heads, plan, layer)
==========================  ================================================

Precondition failures raise ``InvalidArgument`` (a ValueError) with the
reference's message; there is no CPU fallback -- every computation runs in
the CUDA library and a missing library raises ``NativeLibraryError``.
torch is used only for device memory and the current stream.
"""
from __future__ import annotations

import ctypes as C
import math
import threading
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Callable, List, Optional, Sequence

import torch

from . import _lib
from ._lib import InvalidArgument, NativeLibraryError  # noqa: F401  (re-exported)

__all__ = [
    "HeadTensors", "HeadScores", "LayerScores", "TokenSelection", "SparseMode", "ForcedPolicy",
    "SparsePlan", "LayerStat", "score_tokens", "aggregate_scores", "coverage_budget",
    "fixed_budget", "select_tokens", "validate", "dense_causal_attention",
    "token_sparse_attention", "sparse_attention_layer", "InvalidArgument", "NativeLibraryError",
    "rms_norm", "rope_table", "split_heads_rope", "heads_concat", "sparse_attention_layer_host",
    "layer_drift", "select_sparse_layers", "gemm_bf16", "prepare_weight", "row_inv_rms",
    "qkv_proj", "out_proj_residual",
]


# ------------------------------------------------------------------ types
@dataclass
class HeadTensors:
    """attention.hpp:16-25.  q: [H, L, d]; k, v: [Hkv, L, d]; f32 or bf16, CUDA."""

    q: torch.Tensor
    k: torch.Tensor
    v: torch.Tensor

    def __post_init__(self):
        if isinstance(self.q, (list, tuple)):
            self.q = torch.stack(list(self.q))
        if isinstance(self.k, (list, tuple)):
            self.k = torch.stack(list(self.k))
        if isinstance(self.v, (list, tuple)):
            self.v = torch.stack(list(self.v))

    @property
    def n_heads(self) -> int:
        return self.q.shape[0]

    @property
    def n_kv_heads(self) -> int:
        return self.k.shape[0]

    def kv_head(self, h: int) -> int:
        return h // (self.n_heads // self.n_kv_heads)

    @property
    def seq_len(self) -> int:
        return self.q.shape[1]

    @property
    def d_head(self) -> int:
        return self.q.shape[2]


@dataclass
class HeadScores:
    """token_coverage.hpp:12-20."""

    s: torch.Tensor
    last_q: int = 0
    kernel: int = 1


@dataclass
class LayerScores:
    """token_coverage.hpp:23-25."""

    s: torch.Tensor


@dataclass
class TokenSelection:
    """selection.hpp:12-21.  ``indices`` is [H, k_keep] int32 (device), strictly
    ascending per row; internally backed by an [H, L] buffer (C-ABI layout)."""

    indices: torch.Tensor
    k_keep: int = 0
    tau: float = 0.0
    forced: List[int] = field(default_factory=list)
    _full: Optional[torch.Tensor] = field(default=None, repr=False)
    _k_dev: Optional[torch.Tensor] = field(default=None, repr=False)

    def full_buffer(self, seq_len: int) -> torch.Tensor:
        if self._full is None or self._full.shape[1] != seq_len:
            H = self.indices.shape[0]
            buf = torch.zeros((H, seq_len), dtype=torch.int32, device=self.indices.device)
            buf[:, : self.k_keep] = self.indices.to(torch.int32)
            self._full = buf
        return self._full

    def k_device(self) -> torch.Tensor:
        if self._k_dev is None:
            self._k_dev = torch.tensor([self.k_keep], dtype=torch.int32, device=self.indices.device)
        return self._k_dev


class SparseMode(IntEnum):
    """model.hpp:51."""

    kDense = _lib.TSA_MODE_DENSE
    kDynamic = _lib.TSA_MODE_DYNAMIC
    kFixed = _lib.TSA_MODE_FIXED


class ForcedPolicy(IntEnum):
    """model.hpp:54."""

    kFinalToken = _lib.TSA_FORCED_FINAL_TOKEN
    kRecentWindow = _lib.TSA_FORCED_RECENT_WINDOW


@dataclass
class SparsePlan:
    """model.hpp:58-73 (defaults identical)."""

    mode: SparseMode = SparseMode.kDense
    sparse_layers: List[int] = field(default_factory=list)
    tau: float = 0.005
    s_fixed: float = 0.0
    last_q: int = 64
    kernel: int = 7
    forced: ForcedPolicy = ForcedPolicy.kFinalToken

    def check(self, n_layers: int) -> None:
        """model.cpp:47-67."""
        if self.tau < 0.0 or self.tau > 1.0:
            raise InvalidArgument(f"SparsePlan: tau {self.tau:f} outside [0, 1]")
        if self.s_fixed < 0.0 or self.s_fixed >= 1.0:
            raise InvalidArgument(f"SparsePlan: s_fixed {self.s_fixed:f} outside [0, 1)")
        if self.last_q < 1:
            raise InvalidArgument("SparsePlan: last_q must be positive")
        if self.kernel < 1 or self.kernel % 2 == 0:
            raise InvalidArgument("SparsePlan: kernel must be odd and positive")
        for layer in self.sparse_layers:
            if layer < 0 or layer >= n_layers:
                raise InvalidArgument(
                    f"SparsePlan: sparse layer {layer} outside [0, {n_layers})")

    def is_sparse_layer(self, layer: int) -> bool:
        return self.mode != SparseMode.kDense and layer in self.sparse_layers

    def forced_set(self, seq_len: int) -> List[int]:
        """model.cpp:74-79."""
        if self.forced == ForcedPolicy.kFinalToken:
            return [seq_len - 1]
        return list(range(max(0, seq_len - self.last_q), seq_len))


@dataclass
class LayerStat:
    """model.hpp:76-82."""

    layer: int = 0
    sparse: bool = False
    k_keep: int = 0
    attn_flops: float = 0.0
    selection: Optional[TokenSelection] = None


# --------------------------------------------------------------- plumbing
_DTYPES = {torch.float32: _lib.TSA_F32, torch.bfloat16: _lib.TSA_BF16}
_ws_cache: dict = {}


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype not in _DTYPES:
        raise InvalidArgument(f"tsa: unsupported dtype {t.dtype} (float32 or bfloat16)")
    return _DTYPES[t.dtype]


def _require_cuda(*ts: torch.Tensor) -> None:
    for t in ts:
        if not t.is_cuda:
            raise NativeLibraryError(
                "tsa: tensors must live on a CUDA device (the path has no CPU implementation)")


def _ptr(t: Optional[torch.Tensor]):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def _stream(device: torch.device):
    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)


_kd_cache = {}
# Scratch buffers are cached per (device, stream): calls on one stream are
# ordered, so they may share them; calls on different streams (threads) get
# their own -- the operators stay safe to call concurrently.
_cache_lock = threading.Lock()


def _stream_key(device: torch.device):
    return (device.type, device.index, torch.cuda.current_stream(device).cuda_stream)


def _workspace(desc: _lib.TsaDesc, device: torch.device) -> torch.Tensor:
    nbytes = C.c_size_t()
    _lib.check(_lib.load().tsa_workspace_size(C.byref(desc), C.byref(nbytes)))
    key = _stream_key(device)
    with _cache_lock:
        ws = _ws_cache.get(key)
        if ws is None or ws.numel() < nbytes.value:
            ws = torch.zeros(max(nbytes.value, 256), dtype=torch.uint8, device=device)
            _ws_cache[key] = ws
    return ws


def _desc_for(H, Hkv, L, d, dtype, **kw) -> _lib.TsaDesc:
    return _lib.make_desc(H, Hkv, L, d, dtype, **kw)


def _heads_desc(heads: HeadTensors, **kw) -> _lib.TsaDesc:
    _require_cuda(heads.q, heads.k, heads.v)
    q, k, v = heads.q, heads.k, heads.v
    if q.dim() != 3 or k.dim() != 3 or v.dim() != 3:
        raise InvalidArgument("attention: HeadTensors need [heads, L, d] tensors")
    if not (q.dtype == k.dtype == v.dtype):
        raise InvalidArgument("attention: q, k, v dtypes differ")
    H, L, d = q.shape
    Hkv = k.shape[0]
    if k.shape[1:] != (L, d) or v.shape != k.shape:
        raise InvalidArgument(
            f"attention: inconsistent head shapes Q[{L} x {d}] K[{k.shape[1]} x {k.shape[2]}] "
            f"V[{v.shape[1]} x {v.shape[2]}]")
    if Hkv == 0 or H % Hkv != 0:
        raise InvalidArgument(
            f"token_sparse_attention: {H} query heads not divisible by {Hkv} KV heads")
    return _desc_for(H, Hkv, L, d, _dtype_code(q), **kw)


def _contig(*ts):
    return [t.contiguous() for t in ts]


# -------------------------------------------------------------- operators
def score_tokens(heads: HeadTensors, last_q: int, kernel: int, scoring: int = 0) -> HeadScores:
    """token_coverage.cpp:16-50."""
    if last_q < 1:
        raise InvalidArgument(f"score_tokens: last_q must be positive, got {last_q}")
    if kernel < 1 or kernel % 2 == 0:
        raise InvalidArgument(f"avg_pool_1d: kernel must be odd and positive, got {kernel}")
    desc = _heads_desc(heads, last_q=last_q, kernel=kernel, scoring=scoring)
    q, k = _contig(heads.q, heads.k)
    dev = q.device
    s = torch.empty((heads.n_heads, heads.seq_len), dtype=torch.float32, device=dev)
    ws = _workspace(desc, dev)
    _lib.check(_lib.load().tsa_score(C.byref(desc), _ptr(q), _ptr(k), _ptr(s), _ptr(ws), _stream(dev)))
    return HeadScores(s=s, last_q=min(last_q, heads.seq_len), kernel=kernel)


def _scores_desc(s: torch.Tensor, **kw) -> _lib.TsaDesc:
    _require_cuda(s)
    if s.dtype != torch.float32:
        raise InvalidArgument("tsa: scores must be float32")
    H, L = (1, s.shape[0]) if s.dim() == 1 else s.shape
    # geometry of the scores only: d/dtype are placeholders for the workspace
    return _desc_for(H, 1, L, 8, _lib.TSA_F32, last_q=1, **kw)


def aggregate_scores(hs: HeadScores) -> LayerScores:
    """token_coverage.cpp:52-66 (raises on all-zero scores, :62-64)."""
    s = hs.s.contiguous()
    desc = _scores_desc(s)
    dev = s.device
    sl = torch.empty(s.shape[-1], dtype=torch.float32, device=dev)
    ws = _workspace(desc, dev)
    lib = _lib.load()
    _lib.check(lib.tsa_aggregate_scores(C.byref(desc), _ptr(s), _ptr(sl), _ptr(ws), _stream(dev)))
    _lib.check(lib.tsa_check(C.byref(desc), _ptr(ws), _stream(dev)))
    return LayerScores(s=sl)


def coverage_budget(sl: LayerScores, tau: float, min_keep: int) -> int:
    """token_coverage.cpp:68-96 -> k_keep (host int; synchronises)."""
    L = sl.s.shape[0]
    if tau < 0.0 or tau > 1.0:
        raise InvalidArgument(f"coverage_budget: tau {tau:f} outside [0, 1]")
    if min_keep < 1 or min_keep > L:
        raise InvalidArgument(f"coverage_budget: min_keep {min_keep} outside [1, {L}]")
    s = sl.s.contiguous()
    desc = _scores_desc(s, tau=tau)
    dev = s.device
    ws = _workspace(desc, dev)
    k = torch.empty(1, dtype=torch.int32, device=dev)
    _lib.check(_lib.load().tsa_coverage_budget(C.byref(desc), _ptr(s), min_keep, _ptr(k), _ptr(ws),
                                               _stream(dev)))
    return int(k.item())


def fixed_budget(seq_len: int, s: float, min_keep: int) -> int:
    """token_coverage.cpp:98-109 (host integer arithmetic, as in the reference)."""
    if s < 0.0 or s >= 1.0:
        raise InvalidArgument(f"fixed_budget: sparsity ratio {s:f} outside [0, 1)")
    if min_keep < 1 or min_keep > seq_len:
        raise InvalidArgument(f"fixed_budget: min_keep {min_keep} outside [1, {seq_len}]")
    k = int(_lround((1.0 - s) * seq_len))
    return max(k, min_keep)


def _lround(x: float) -> int:
    return int(math.floor(x + 0.5)) if x >= 0 else -int(math.floor(-x + 0.5))


def _normalize_forced(forced: Sequence[int], L: int) -> List[int]:
    f = sorted(set(int(t) for t in forced))
    for t in f:
        if t < 0 or t >= L:
            raise InvalidArgument(f"select_tokens: forced index {t} out of range [0, {L})")
    return f


def select_tokens(hs: HeadScores, k_keep: int, forced: Sequence[int] = ()) -> TokenSelection:
    """token_coverage.cpp:111-152."""
    s = hs.s.contiguous()
    _require_cuda(s)
    H, L = s.shape
    f = _normalize_forced(forced, L)
    min_keep = max(1, len(f))
    if k_keep < min_keep or k_keep > L:
        raise InvalidArgument(f"select_tokens: k_keep {k_keep} outside [{min_keep}, {L}]")
    desc = _scores_desc(s)
    dev = s.device
    ws = _workspace(desc, dev)
    idx = torch.empty((H, L), dtype=torch.int32, device=dev)
    kd = torch.tensor([k_keep], dtype=torch.int32, device=dev)
    fd = torch.tensor(f if f else [0], dtype=torch.int32, device=dev)
    _lib.check(_lib.load().tsa_select(C.byref(desc), _ptr(s), _ptr(kd), _ptr(fd), len(f),
                                      _ptr(idx), None, _ptr(ws), _stream(dev)))
    return TokenSelection(indices=idx[:, :k_keep], k_keep=k_keep, forced=f, _full=idx, _k_dev=kd)


def validate(sel: TokenSelection, seq_len: int) -> None:
    """selection.cpp:12-45 (host check of a selection)."""
    min_keep = max(1, len(sel.forced))
    if sel.k_keep < min_keep or sel.k_keep > seq_len:
        raise InvalidArgument(
            f"validate: k_keep {sel.k_keep} outside [{min_keep}, {seq_len}]")
    idx = sel.indices.detach().to("cpu", torch.int64)
    for h in range(idx.shape[0]):
        row = idx[h].tolist()
        if len(row) != sel.k_keep:
            raise InvalidArgument(
                f"validate: head {h} keeps {len(row)} tokens, expected {sel.k_keep}")
        for r, t in enumerate(row):
            if t < 0 or t >= seq_len:
                raise InvalidArgument(
                    f"validate: head {h} index {t} out of range [0, {seq_len})")
            if r > 0 and t <= row[r - 1]:
                raise InvalidArgument(
                    f"validate: head {h} indices not strictly ascending at position {r}")
        present = set(row)
        for f in sel.forced:
            if f not in present:
                raise InvalidArgument(f"validate: head {h} is missing forced index {f}")


def dense_causal_attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor) -> torch.Tensor:
    """attention.cpp:25-40 for one head: [n, d] -> [n, d]."""
    if q.shape[1] != k.shape[1] or k.shape[0] != v.shape[0] or k.shape[1] != q.shape[1]:
        raise InvalidArgument(
            f"attention: inconsistent head shapes Q[{q.shape[0]} x {q.shape[1]}] "
            f"K[{k.shape[0]} x {k.shape[1]}] V[{v.shape[0]} x {v.shape[1]}]")
    if q.shape[0] != k.shape[0]:
        raise InvalidArgument(
            f"dense_causal_attention: Q[{q.shape[0]} x {q.shape[1]}] and "
            f"K[{k.shape[0]} x {k.shape[1]}] disagree on length")
    heads = HeadTensors(q.unsqueeze(0), k.unsqueeze(0), v.unsqueeze(0))
    desc = _heads_desc(heads)
    qq, kk, vv = _contig(heads.q, heads.k, heads.v)
    out = torch.empty_like(qq)
    dev = qq.device
    _lib.check(_lib.load().tsa_dense_attention(C.byref(desc), _ptr(qq), _ptr(kk), _ptr(vv),
                                               _ptr(out), _stream(dev)))
    return out[0]


AttentionKernel = Callable[[torch.Tensor, torch.Tensor, torch.Tensor], torch.Tensor]


def token_sparse_attention(heads: HeadTensors, sel: TokenSelection,
                           inner: Optional[AttentionKernel] = None,
                           check_selection: bool = True) -> torch.Tensor:
    """attention.cpp:74-99.  Returns [H, L, d].

    ``inner`` is the AttentionKernel seam (attention.hpp:28): None runs the
    library's causal kernel (tcgen05 for bf16/d=128); a callable is invoked
    once per head with the compressed [k, d] Q^/K^/V^ (the contract pinned by
    test_attention.cpp:318-338) and must return [k, d]."""
    desc = _heads_desc(heads)
    H, L = heads.n_heads, heads.seq_len
    if sel.indices.shape[0] != H:
        raise InvalidArgument(
            f"token_sparse_attention: selection covers {sel.indices.shape[0]} heads, "
            f"tensors have {H}")
    if check_selection:
        validate(sel, L)
    q, k, v = _contig(heads.q, heads.k, heads.v)
    dev = q.device
    ws = _workspace(desc, dev)
    idx = sel.full_buffer(L)
    kd = sel.k_device()
    out = torch.empty_like(q)
    lib = _lib.load()
    st = _stream(dev)
    if inner is None:
        _lib.check(lib.tsa_token_sparse_attention(C.byref(desc), _ptr(q), _ptr(k), _ptr(v),
                                                  _ptr(idx), _ptr(kd), _ptr(out), _ptr(ws), st))
        return out
    qc, kc, vc, oc = (torch.empty_like(q) for _ in range(4))
    _lib.check(lib.tsa_gather(C.byref(desc), _ptr(q), _ptr(k), _ptr(v), _ptr(idx), _ptr(kd),
                              _ptr(qc), _ptr(kc), _ptr(vc), st))
    n = sel.k_keep
    for h in range(H):
        oc[h, :n] = inner(qc[h, :n], kc[h, :n], vc[h, :n])
    _lib.check(lib.tsa_scatter_rows(C.byref(desc), _ptr(oc), _ptr(idx), _ptr(kd), _ptr(out),
                                    _ptr(ws), st))
    return out


def sparse_attention_layer(heads: HeadTensors, plan: SparsePlan, layer: int = 0,
                           out: Optional[torch.Tensor] = None, stat: bool = True,
                           scoring: int = 0):
    """The attention branch of layer_forward (model.cpp:169-195) for one layer.

    Sparse layers run score -> budget -> select -> gather -> attend -> scatter
    in one C-ABI call; dense layers run the causal kernel on every head.
    Returns (out [H, L, d], LayerStat)."""
    L = heads.seq_len
    sparse = plan.is_sparse_layer(layer)
    mode = plan.mode if sparse else SparseMode.kDense
    desc = _heads_desc(heads, mode=int(mode), tau=plan.tau, s_fixed=plan.s_fixed,
                       last_q=plan.last_q, kernel=plan.kernel, forced_policy=int(plan.forced),
                       scoring=scoring)
    q, k, v = _contig(heads.q, heads.k, heads.v)
    dev = q.device
    ws = _workspace(desc, dev)
    if out is None:
        out = torch.empty_like(q)
    if stat:  # the caller keeps the selection: fresh buffers
        idx = torch.empty((heads.n_heads, L), dtype=torch.int32, device=dev) if sparse else None
        kd = torch.empty(1, dtype=torch.int32, device=dev)
    else:  # selection stays in the workspace; stable addresses keep the graph cache warm
        idx = None
        key = _stream_key(dev)
        with _cache_lock:
            kd = _kd_cache.get(key)
            if kd is None:
                kd = _kd_cache[key] = torch.empty(1, dtype=torch.int32, device=dev)
    _lib.check(_lib.load().tsa_sparse_attention_layer(
        C.byref(desc), _ptr(q), _ptr(k), _ptr(v), _ptr(out), _ptr(idx), _ptr(kd), None,
        _ptr(ws), _stream(dev)))
    if not stat:
        return out, None
    k_keep = int(kd.item())
    st = LayerStat(layer=layer, sparse=sparse, k_keep=k_keep,
                   attn_flops=4.0 * k_keep * k_keep * heads.d_head * heads.n_heads)
    if sparse:
        st.selection = TokenSelection(indices=idx[:, :k_keep], k_keep=k_keep,
                                      tau=plan.tau if plan.mode == SparseMode.kDynamic else 0.0,
                                      forced=plan.forced_set(L), _full=idx, _k_dev=kd)
    return out, st


# ------------------------------------------- attention-branch producer / consumer
def rms_norm(x: torch.Tensor, gain: torch.Tensor, eps: float,
             out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """model.cpp:81-94 over the rows of x [rows, cols] (f32 or bf16, CUDA)."""
    _require_cuda(x, gain)
    if x.dim() != 2:
        raise InvalidArgument("rms_norm: x must be [rows, cols]")
    if gain.numel() != x.shape[1]:
        raise InvalidArgument(f"rms_norm: gain size {gain.numel()} != width of "
                              f"[{x.shape[0]} x {x.shape[1]}]")
    x = x.contiguous()
    g = gain.to(torch.float32).contiguous()
    if out is None:
        out = torch.empty_like(x)
    _lib.check(_lib.load().tsa_rms_norm(_ptr(x), _ptr(g), x.shape[0], x.shape[1], eps,
                                        _dtype_code(x), _ptr(out), _stream(x.device)))
    return out


def rope_table(seq_len: int, d_head: int, theta: float, device) -> torch.Tensor:
    """apply_rope's (cos, sin) at positions 0..L-1 (model.cpp:107-116): f32 [L, d/2, 2]."""
    t = torch.empty((seq_len, d_head // 2, 2), dtype=torch.float32, device=device)
    _lib.check(_lib.load().tsa_rope_table(seq_len, d_head, theta, _ptr(t),
                                          _stream(torch.device(device))))
    return t


def split_heads_rope(qkv: torch.Tensor, table: torch.Tensor, n_heads: int, n_kv_heads: int,
                     d_head: int, out: Optional[HeadTensors] = None) -> HeadTensors:
    """split_heads + apply_rope of project_qkv (model.cpp:128-158): projection rows
    [L, (H + 2 Hkv) d] -> HeadTensors with RoPE on q and k."""
    _require_cuda(qkv, table)
    L = qkv.shape[0]
    if qkv.shape[1] != (n_heads + 2 * n_kv_heads) * d_head:
        raise InvalidArgument("split_heads_rope: projection width != (H + 2 Hkv) d")
    if out is None:
        out = HeadTensors(torch.empty((n_heads, L, d_head), dtype=qkv.dtype, device=qkv.device),
                          torch.empty((n_kv_heads, L, d_head), dtype=qkv.dtype, device=qkv.device),
                          torch.empty((n_kv_heads, L, d_head), dtype=qkv.dtype, device=qkv.device))
    desc = _desc_for(n_heads, n_kv_heads, L, d_head, _dtype_code(qkv))
    qkv = qkv.contiguous()
    _lib.check(_lib.load().tsa_split_heads_rope(C.byref(desc), _ptr(qkv), _ptr(table),
                                                _ptr(out.q), _ptr(out.k), _ptr(out.v),
                                                _stream(qkv.device)))
    return out


def heads_concat(heads: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """model.cpp:196-200: [H, L, d] -> [L, H d]."""
    _require_cuda(heads)
    H, L, d = heads.shape
    heads = heads.contiguous()
    if out is None:
        out = torch.empty((L, H * d), dtype=heads.dtype, device=heads.device)
    desc = _desc_for(H, H, L, d, _dtype_code(heads))
    _lib.check(_lib.load().tsa_heads_concat(C.byref(desc), _ptr(heads), _ptr(out),
                                            _stream(heads.device)))
    return out


# ---- the projections on the tensor cores (proj_gemm.cu)
def gemm_bf16(a: torch.Tensor, b_t: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """c [M, N] = a [M, K] b_t[N, K]^T on the hand-written tcgen05 GEMM (bf16,
    f32 accumulation; N % 256 == 0, K % 64 == 0)."""
    _require_cuda(a, b_t)
    if a.dtype != torch.bfloat16 or b_t.dtype != torch.bfloat16:
        raise InvalidArgument("gemm_bf16: a and b_t must be bf16")
    M, K = a.shape
    N = b_t.shape[0]
    if b_t.shape[1] != K:
        raise InvalidArgument(f"gemm_bf16: inner dimensions differ ({K} vs {b_t.shape[1]})")
    a, b_t = a.contiguous(), b_t.contiguous()
    if out is None:
        out = torch.empty((M, N), dtype=torch.bfloat16, device=a.device)
    _lib.check(_lib.load().tsa_gemm_bf16(_ptr(a), _ptr(b_t), _ptr(out), M, N, K,
                                         _stream(a.device)))
    return out


def prepare_weight(w: torch.Tensor, gain: Optional[torch.Tensor] = None) -> torch.Tensor:
    """The projections' weight layout, once per weight: (diag(gain) w)^T as bf16
    [cols, rows] for w [rows, cols] (f32 or bf16).  W_qkv takes the attention
    norm's gain (rms_norm folds into the weight), W_o none."""
    _require_cuda(w)
    rows, cols = w.shape
    w = w.contiguous()
    g = None
    if gain is not None:
        if gain.numel() != rows:
            raise InvalidArgument(f"prepare_weight: gain size {gain.numel()} != {rows} rows")
        g = gain.to(torch.float32).contiguous()
    out = torch.empty((cols, rows), dtype=torch.bfloat16, device=w.device)
    _lib.check(_lib.load().tsa_prepare_weight(_ptr(w), _dtype_code(w), _ptr(g) if g is not None
                                              else None, rows, cols, _ptr(out), _stream(w.device)))
    return out


def row_inv_rms(x: torch.Tensor, eps: float, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """rms_norm's row statistic (model.cpp:81-94): 1 / sqrt(mean_j x^2 + eps), f32 [rows]."""
    _require_cuda(x)
    if x.dtype != torch.bfloat16 or x.dim() != 2:
        raise InvalidArgument("row_inv_rms: x must be bf16 [rows, cols]")
    x = x.contiguous()
    if out is None:
        out = torch.empty(x.shape[0], dtype=torch.float32, device=x.device)
    _lib.check(_lib.load().tsa_row_inv_rms(_ptr(x), x.shape[0], x.shape[1], eps, _ptr(out),
                                           _stream(x.device)))
    return out


def qkv_proj(x: torch.Tensor, w_t: torch.Tensor, inv_rms: Optional[torch.Tensor],
             table: torch.Tensor, n_heads: int, n_kv_heads: int, d_head: int,
             out: Optional[HeadTensors] = None) -> HeadTensors:
    """project_qkv with rms_norm folded in (model.cpp:81-94, 128-158), one tcgen05
    GEMM: q / k / v heads of rope((inv_rms * x) W') with w_t = prepare_weight(W_qkv,
    gain) and the RoPE table of rope_table."""
    _require_cuda(x, w_t, table)
    L, D = x.shape
    if w_t.shape != ((n_heads + 2 * n_kv_heads) * d_head, D):
        raise InvalidArgument("qkv_proj: w_t must be [(H + 2 Hkv) d, d_model]")
    if x.dtype != torch.bfloat16 or w_t.dtype != torch.bfloat16:
        raise InvalidArgument("qkv_proj: x and w_t must be bf16")
    if inv_rms is not None and (inv_rms.dtype != torch.float32 or inv_rms.numel() < L):
        raise InvalidArgument("qkv_proj: inv_rms must be f32 [L]")
    if out is None:
        out = HeadTensors(torch.empty((n_heads, L, d_head), dtype=x.dtype, device=x.device),
                          torch.empty((n_kv_heads, L, d_head), dtype=x.dtype, device=x.device),
                          torch.empty((n_kv_heads, L, d_head), dtype=x.dtype, device=x.device))
    desc = _desc_for(n_heads, n_kv_heads, L, d_head, _dtype_code(x))
    x = x.contiguous()
    _lib.check(_lib.load().tsa_qkv_proj(C.byref(desc), _ptr(x), D, _ptr(w_t),
                                        _ptr(inv_rms) if inv_rms is not None else None,
                                        _ptr(table), _ptr(out.q), _ptr(out.k), _ptr(out.v),
                                        _stream(x.device)))
    return out


def out_proj_residual(o: torch.Tensor, wo_t: torch.Tensor, x: torch.Tensor) -> torch.Tensor:
    """x += concat_h(o_h) W_o in place (model.cpp:196-201), A read from o [H, L, d]
    directly; wo_t = prepare_weight(W_o)."""
    _require_cuda(o, wo_t, x)
    H, L, d = o.shape
    D = x.shape[1]
    if x.shape[0] != L or wo_t.shape != (D, H * d):
        raise InvalidArgument("out_proj_residual: shapes do not match")
    if o.dtype != torch.bfloat16 or wo_t.dtype != torch.bfloat16 or x.dtype != torch.bfloat16:
        raise InvalidArgument("out_proj_residual: o, wo_t and x must be bf16")
    if not (o.is_contiguous() and x.is_contiguous()):
        raise InvalidArgument("out_proj_residual: o and x must be contiguous")
    desc = _desc_for(H, H, L, d, _dtype_code(o))
    _lib.check(_lib.load().tsa_out_proj_residual(C.byref(desc), _ptr(o), _ptr(wo_t), D, _ptr(x),
                                                 _stream(o.device)))
    return x


_staging: dict = {}


def sparse_attention_layer_host(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor,
                                out: torch.Tensor, plan: SparsePlan, device=None,
                                n_groups: int = 0, scoring: int = 0,
                                overlap: bool = True) -> torch.Tensor:
    """The sparse layer on HOST tensors (the reference's calling convention):
    q [H, L, d], k / v [Hkv, L, d] and out [H, L, d] in (pinned) host memory.
    Transfers are pipelined with the compute (tsa_sparse_attention_layer_host);
    returns the device k_keep (int32[1]); ``out`` is complete once the current
    stream of ``device`` has drained.

    overlap (default): consecutive calls alternate between two device staging
    sets, each on its own stream, so a call's K copy and scoring overlap the
    previous call's attention (the copies of one call only wait for the call
    before the last, which used the same buffers).  The returned k_keep stays
    valid until the call after next."""
    device = torch.device(device or "cuda")
    for t in (q, k, v, out):
        if t.is_cuda:
            raise InvalidArgument("sparse_attention_layer_host: q, k, v, out must be host tensors")
    H, L, d = q.shape
    Hkv = k.shape[0]
    desc = _desc_for(H, Hkv, L, d, _dtype_code(q), mode=int(plan.mode), tau=plan.tau,
                     s_fixed=plan.s_fixed, last_q=plan.last_q, kernel=plan.kernel,
                     forced_policy=int(plan.forced), scoring=scoring)
    key = _stream_key(device) + (q.dtype, H, Hkv, L, d, bool(overlap))
    with _cache_lock:
        ent = _staging.get(key)
        if ent is None:
            sets = []
            for _ in range(2 if overlap else 1):
                side = torch.cuda.Stream(device) if overlap else None
                sets.append((side, (
                    torch.empty_like(q, device=device), torch.empty_like(k, device=device),
                    torch.empty_like(v, device=device), torch.empty_like(out, device=device),
                    torch.empty(1, dtype=torch.int32, device=device))))
            ent = _staging[key] = [0, sets]
        i = ent[0]
        ent[0] = (i + 1) % len(ent[1])
        side, bufs = ent[1][i]
    qd, kd, vd, od, kk = bufs
    cur = torch.cuda.current_stream(device)
    with torch.cuda.stream(side if side is not None else cur):
        ws = _workspace(desc, device)  # per stream: each staging set has its own
        _lib.check(_lib.load().tsa_sparse_attention_layer_host(
            C.byref(desc), _ptr(q), _ptr(k), _ptr(v), _ptr(out), _ptr(qd), _ptr(kd), _ptr(vd),
            _ptr(od), None, _ptr(kk), None, _ptr(ws), n_groups, _stream(device)))
    if side is not None:
        cur.wait_stream(side)  # `out` complete once the caller's stream drains
    return kk


# ------------------------------------------------------------ drift calibration
def layer_drift(prev: torch.Tensor, nxt: torch.Tensor, epsilon: float = 1e-6,
                out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """compute_drift (drift.cpp:14-45) for one layer boundary: the mean over rows
    of |next - prev| / (|prev| + eps), in double; returns a device float64 [1]
    (written asynchronously, no host sync)."""
    _require_cuda(prev, nxt)
    if prev.shape != nxt.shape or prev.dim() != 2 or prev.dtype != nxt.dtype:
        raise InvalidArgument(f"compute_drift: shape {tuple(nxt.shape)} != {tuple(prev.shape)}")
    prev, nxt = prev.contiguous(), nxt.contiguous()
    if out is None:
        out = torch.empty(1, dtype=torch.float64, device=prev.device)
    ws = torch.empty(prev.shape[0], dtype=torch.float64, device=prev.device)
    _lib.check(_lib.load().tsa_layer_drift(_ptr(prev), _ptr(nxt), prev.shape[0], prev.shape[1],
                                           _dtype_code(prev), epsilon, _ptr(out), _ptr(ws),
                                           _stream(prev.device)))
    return out


def select_sparse_layers(R: Sequence[float], delta: float):
    """drift.cpp:47-65: (R_hat, sparse layers) with R_hat[l] = #{k: R[k] <= R[l]} / n."""
    r = (C.c_double * len(R))(*[float(x) for x in R])
    rh = (C.c_double * len(R))()
    layers = (C.c_int32 * len(R))()
    m = C.c_int32()
    _lib.check(_lib.load().tsa_select_sparse_layers(r, len(R), delta, rh, layers, C.byref(m)))
    return list(rh), list(layers[:m.value])
