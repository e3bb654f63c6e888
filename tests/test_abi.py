"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/tsa_b200.h declares, and host-side validation reports the
reference's error wording."""
import ctypes as C
import re
from pathlib import Path

import pytest

from paper_2602_03216_b200 import _lib

ROOT = Path(__file__).resolve().parent.parent


def header_symbols():
    text = (ROOT / "include" / "tsa_b200.h").read_text()
    return sorted(set(re.findall(r"TSA_API\s+[\w\s\*]+?\b(tsa_\w+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 15
    for name in syms:
        assert hasattr(lib, name), name
    assert sorted(_lib.EXPORTS) == syms


def test_library_is_sm100a_cubin():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_lib.LIB_PATH)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_desc_defaults_follow_sparse_plan():
    d = _lib.make_desc(32, 8, 4096, 128, _lib.TSA_BF16)
    # SparsePlan defaults, model.hpp:58-73
    assert (d.tau, d.s_fixed, d.last_q, d.kernel) == (0.005, 0.0, 64, 7)
    assert d.forced_policy == _lib.TSA_FORCED_FINAL_TOKEN
    assert (d.head_begin, d.head_end) == (0, 32)


@pytest.mark.parametrize("field,value,msg", [
    ("n_kv_heads", 3, "query heads not divisible by 3 KV heads"),
    ("last_q", 0, "score_tokens: last_q must be positive, got 0"),
    ("kernel", 4, "avg_pool_1d: kernel must be odd and positive, got 4"),
    ("tau", 1.5, "coverage_budget: tau 1.500000 outside [0, 1]"),
    ("s_fixed", 1.0, "fixed_budget: sparsity ratio 1.000000 outside [0, 1)"),
    ("d_head", 300, "unsupported d_head 300"),
    ("head_end", 3, "splits a KV group"),
])
def test_validation_messages(field, value, msg):
    lib = _lib.load()
    d = _lib.make_desc(32, 8, 1024, 128, _lib.TSA_BF16)
    setattr(d, field, value)
    n = C.c_size_t()
    rc = lib.tsa_workspace_size(C.byref(d), C.byref(n))
    assert rc == _lib.TSA_ERR_INVALID
    assert msg in lib.tsa_last_error().decode()
    with pytest.raises(_lib.InvalidArgument, match=re.escape(msg)):
        _lib.check(rc)


def test_workspace_size_scales_with_geometry():
    lib = _lib.load()
    n1, n2 = C.c_size_t(), C.c_size_t()
    lib.tsa_workspace_size(C.byref(_lib.make_desc(32, 8, 4096, 128, _lib.TSA_BF16)), C.byref(n1))
    lib.tsa_workspace_size(C.byref(_lib.make_desc(32, 8, 8192, 128, _lib.TSA_BF16)), C.byref(n2))
    assert n2.value > 1.9 * n1.value


def test_cpu_tensors_fail_loudly():
    import torch
    from paper_2602_03216_b200 import HeadTensors, NativeLibraryError, score_tokens
    h = HeadTensors(torch.zeros(2, 8, 8), torch.zeros(1, 8, 8), torch.zeros(1, 8, 8))
    with pytest.raises(NativeLibraryError):
        score_tokens(h, 4, 1)
