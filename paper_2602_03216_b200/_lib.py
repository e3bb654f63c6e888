"""ctypes binding of the C ABI (include/tsa_b200.h) -> ``libtsa_b200.so``.

The library is built in-tree by ``paper_2602_03216_b200/build.py`` (nvcc,
sm_100a).  There is no fallback: if the shared library is missing or cannot
be loaded, every operation raises ``NativeLibraryError``.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libtsa_b200.so"

TSA_F32, TSA_BF16 = 0, 1
TSA_MODE_DENSE, TSA_MODE_DYNAMIC, TSA_MODE_FIXED = 0, 1, 2
TSA_FORCED_FINAL_TOKEN, TSA_FORCED_RECENT_WINDOW = 0, 1
TSA_SCORING_DEFAULT, TSA_SCORING_REFERENCE, TSA_SCORING_FAST = 0, 1, 2
TSA_OK, TSA_ERR_INVALID, TSA_ERR_CUDA, TSA_ERR_NCCL = 0, 1, 2, 3

# Every symbol include/tsa_b200.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "tsa_desc_init", "tsa_last_error", "tsa_version", "tsa_kernel_launches", "tsa_release_graphs", "tsa_workspace_size", "tsa_score",
    "tsa_budget", "tsa_aggregate_scores", "tsa_coverage_budget", "tsa_select", "tsa_gather",
    "tsa_attend", "tsa_attend_indexed", "tsa_zero_unselected", "tsa_gather_zero", "tsa_scatter",
    "tsa_scatter_rows", "tsa_check", "tsa_token_sparse_attention",
    "tsa_dense_attention", "tsa_sparse_attention_layer", "tsa_rms_norm", "tsa_rope_table",
    "tsa_split_heads_rope", "tsa_heads_concat", "tsa_sparse_attention_layer_host",
    "tsa_layer_drift", "tsa_select_sparse_layers", "tsa_gather_zero_replicas",
    "tsa_attend_indexed_replicas", "tsa_score_replicas", "tsa_ipc_alloc", "tsa_ipc_open",
    "tsa_ipc_close", "tsa_ipc_free", "tsa_peer_barrier", "tsa_expf", "tsa_peer_check",
    "tsa_sparse_attention_layer_sharded", "tsa_gemm_bf16", "tsa_prepare_weight",
    "tsa_row_inv_rms", "tsa_qkv_proj", "tsa_out_proj_residual",
)
TSA_IPC_HANDLE_BYTES = 64
TSA_MAX_REPLICAS = 8


class NativeLibraryError(RuntimeError):
    """The CUDA library is missing or unusable (no CPU fallback exists)."""


class InvalidArgument(ValueError):
    """Precondition failure -- the reference throws std::invalid_argument here."""


class CudaError(RuntimeError):
    pass


class TsaDesc(C.Structure):
    _fields_ = [
        ("n_heads", C.c_int32), ("n_kv_heads", C.c_int32), ("seq_len", C.c_int32),
        ("d_head", C.c_int32), ("dtype", C.c_int32), ("mode", C.c_int32),
        ("tau", C.c_double), ("s_fixed", C.c_double), ("last_q", C.c_int32),
        ("kernel", C.c_int32), ("forced_policy", C.c_int32), ("head_begin", C.c_int32),
        ("head_end", C.c_int32), ("scoring", C.c_int32),
    ]


_lib = None


def load() -> C.CDLL:
    """Load libtsa_b200.so (building it first if this is a build container)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        try:
            from . import build as _build
            _build.build()
        except Exception as e:  # pragma: no cover - depends on toolchain
            raise NativeLibraryError(f"{LIB_PATH} is missing and could not be built: {e}") from e
    try:
        lib = C.CDLL(str(LIB_PATH))
    except OSError as e:
        raise NativeLibraryError(f"cannot load {LIB_PATH}: {e}") from e
    P, I, D = C.c_void_p, C.c_int32, C.POINTER(TsaDesc)
    sig = {
        "tsa_desc_init": (None, [D, I, I, I, I, I]),
        "tsa_last_error": (C.c_char_p, []),
        "tsa_version": (C.c_char_p, []),
        "tsa_kernel_launches": (C.c_uint64, []),
        "tsa_release_graphs": (None, []),
        "tsa_rms_norm": (C.c_int, [P, P, C.c_int64, I, C.c_float, I, P, P]),
        "tsa_rope_table": (C.c_int, [I, I, C.c_float, P, P]),
        "tsa_split_heads_rope": (C.c_int, [D, P, P, P, P, P, P]),
        "tsa_heads_concat": (C.c_int, [D, P, P, P]),
        "tsa_gemm_bf16": (C.c_int, [P, P, P, I, I, I, P]),
        "tsa_prepare_weight": (C.c_int, [P, I, P, I, I, P, P]),
        "tsa_row_inv_rms": (C.c_int, [P, C.c_int64, I, C.c_float, P, P]),
        "tsa_qkv_proj": (C.c_int, [D, P, I, P, P, P, P, P, P, P]),
        "tsa_out_proj_residual": (C.c_int, [D, P, P, I, P, P]),
        "tsa_layer_drift": (C.c_int, [P, P, C.c_int64, I, I, C.c_double, P, P, P]),
        "tsa_select_sparse_layers": (C.c_int, [P, I, C.c_double, P, P, P]),
        "tsa_sparse_attention_layer_host": (C.c_int, [D, P, P, P, P, P, P, P, P, P, P, P, P, I, P]),
        "tsa_workspace_size": (C.c_int, [D, C.POINTER(C.c_size_t)]),
        "tsa_score": (C.c_int, [D, P, P, P, P, P]),
        "tsa_expf": (C.c_int, [P, P, C.c_int64, P]),
        "tsa_budget": (C.c_int, [D, P, P, P, P]),
        "tsa_aggregate_scores": (C.c_int, [D, P, P, P, P]),
        "tsa_coverage_budget": (C.c_int, [D, P, I, P, P, P]),
        "tsa_select": (C.c_int, [D, P, P, P, I, P, P, P, P]),
        "tsa_gather": (C.c_int, [D, P, P, P, P, P, P, P, P, P]),
        "tsa_attend": (C.c_int, [D, P, P, P, P, I, P, P]),
        "tsa_scatter": (C.c_int, [D, P, P, P, P]),
        "tsa_attend_indexed": (C.c_int, [D, P, P, P, P, P, P, P, P, P]),
        "tsa_zero_unselected": (C.c_int, [D, P, P, P]),
        "tsa_gather_zero": (C.c_int, [D, P, P, P, P, P, P, P, P, P]),
        "tsa_gather_zero_replicas": (C.c_int, [D, P, P, P, P, P, P, P, P, I, P]),
        "tsa_score_replicas": (C.c_int, [D, P, P, P, I, P, P]),
        "tsa_ipc_alloc": (C.c_int, [C.c_size_t, C.POINTER(C.c_void_p), P]),
        "tsa_ipc_open": (C.c_int, [P, C.POINTER(C.c_void_p)]),
        "tsa_ipc_close": (C.c_int, [P]),
        "tsa_ipc_free": (C.c_int, [P]),
        "tsa_peer_barrier": (C.c_int, [P, I, I, I, P]),
        "tsa_peer_check": (C.c_int, [P, I, I, P]),
        "tsa_sparse_attention_layer_sharded": (C.c_int, [D, P, P, P, P, P, P, P, P, P, P]),
        "tsa_attend_indexed_replicas": (C.c_int, [D, P, P, P, P, P, P, P, P, I, P]),
        "tsa_scatter_rows": (C.c_int, [D, P, P, P, P, P, P]),
        "tsa_check": (C.c_int, [D, P, P]),
        "tsa_token_sparse_attention": (C.c_int, [D, P, P, P, P, P, P, P, P]),
        "tsa_dense_attention": (C.c_int, [D, P, P, P, P, P]),
        "tsa_sparse_attention_layer": (C.c_int, [D, P, P, P, P, P, P, P, P, P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int) -> None:
    if rc == TSA_OK:
        return
    msg = load().tsa_last_error().decode()
    if rc == TSA_ERR_INVALID:
        raise InvalidArgument(msg)
    raise CudaError(msg)


def make_desc(n_heads, n_kv_heads, seq_len, d_head, dtype, **kw) -> TsaDesc:
    d = TsaDesc()
    load().tsa_desc_init(C.byref(d), n_heads, n_kv_heads, seq_len, d_head, dtype)
    for k, v in kw.items():
        if v is not None:
            setattr(d, k, v)
    return d
