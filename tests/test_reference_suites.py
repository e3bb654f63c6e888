"""The reference's OWN hot-path unit suites (proj/tests/test_attention.cpp,
test_coverage.cpp -- compiled unmodified) linked against the B200 adapter, so
every reference test case exercises the CUDA path.  Built by oracle/Makefile
(`make gpu-suites`) in the build container; run on the GPU box."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
SUITES = ["gpu_test_coverage", "gpu_test_attention"]


@pytest.mark.gpu
@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_on_b200(cuda, suite):
    exe = ROOT / "oracle" / "_ref" / suite
    if not exe.exists():
        pytest.fail(f"{exe} not built (run python __graft_entry__.py in the build container)")
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    print(r.stdout[-2000:], r.stderr[-4000:])
    assert r.returncode == 0, r.stderr[-4000:]
    assert "failed: 0" in r.stdout


def test_reference_suites_link_the_b200_library():
    """The suite binaries resolve the operators from libtsa_b200.so (CPU-side check)."""
    for suite in SUITES:
        exe = ROOT / "oracle" / "_ref" / suite
        if not exe.exists():
            pytest.skip("suites not built")
        out = subprocess.run(["ldd", str(exe)], capture_output=True, text=True).stdout
        assert "libtsa_b200.so" in out
        syms = subprocess.run(["nm", "-C", str(exe)], capture_output=True, text=True).stdout
        # the operator definitions come from the adapter, not the reference's sources
        assert "tsa::score_tokens" in syms and "ref_cpu_token_sparse_attention" in syms


def test_reference_model_suite_pins_the_shim():
    """proj/tests/test_model.cpp (rms_norm, apply_rope, project_qkv, layer_forward,
    init_random, checkpoints) compiled unmodified against the Eigen/doctest shim:
    pins model.cpp's arithmetic that the producer oracle restates (CPU)."""
    exe = ROOT / "oracle" / "_ref" / "test_model"
    if not exe.exists():
        pytest.skip("reference suites not built")
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "failed: 0" in r.stdout
