"""Codegen guards for the tcgen05 attention kernel (CPU: cuobjdump on the
built library).  The MMA warp must issue UTCHMMA from uniform registers --
when the kernel's other roles grow, ptxas can move the TMEM addresses into
vector registers and every TS-MMA then pays an R2UR.BROADCAST (measured 2-4 %
on the 128K layer) -- and nothing may spill to local memory."""
import re
import shutil
import subprocess
from pathlib import Path

import pytest

LIB = Path(__file__).resolve().parent.parent / "paper_2602_03216_b200" / "libtsa_b200.so"
CUOBJDUMP = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"


@pytest.fixture(scope="module")
def attend_sass():
    if not LIB.exists() or not Path(CUOBJDUMP).exists():
        pytest.skip("library not built or cuobjdump absent")
    txt = subprocess.run([CUOBJDUMP, "-sass", str(LIB)], capture_output=True, text=True,
                         check=True).stdout
    out = {}
    for part in re.split(r"\n\s*Function : ", txt):
        name = part.split("\n", 1)[0]
        # the default instantiation: a quarter of the exponentials on the FMA pipe
        m = re.search(r"attend_sm100_kernelILb([01])ELj4369EE", name)
        if m:
            out["indexed" if m.group(1) == "1" else "dense"] = part
    assert set(out) == {"indexed", "dense"}, list(out)
    return out


@pytest.mark.parametrize("kind", ["dense", "indexed"])
def test_attention_sass_uses_tcgen05_and_tma(attend_sass, kind):
    s = attend_sass[kind]
    assert s.count("UTCHMMA") >= 48          # S (SS) and PV (TS) MMAs, unrolled
    assert "UTMALDG" in s and "LDTM" in s and "STTM" in s
    if kind == "indexed":
        assert "UTMALDG.2D.GATHER4" in s     # Q rows by TMA gather4


@pytest.mark.parametrize("kind", ["dense", "indexed"])
def test_attention_mma_operands_stay_uniform(attend_sass, kind):
    s = attend_sass[kind]
    assert "LDL" not in s and "STL" not in s  # no spills
    # the only broadcasts are the gather4 issue loop's (indexed: 10 row indices)
    assert s.count("R2UR.BROADCAST") <= (12 if kind == "indexed" else 0)
    assert s.count("R2UR ") <= 16


def test_projection_gemm_sass_is_2cta_tcgen05():
    """proj_gemm.cu: every instantiation issues cta_group::2 MMAs
    (UTCHMMA.2CTA) fed by pair TMA loads (UTMALDG.*.2CTA), reads the
    accumulator with LDTM, and does not spill."""
    if not LIB.exists() or not Path(CUOBJDUMP).exists():
        pytest.skip("library not built or cuobjdump absent")
    txt = subprocess.run([CUOBJDUMP, "-sass", str(LIB)], capture_output=True, text=True,
                         check=True).stdout
    parts = [p for p in re.split(r"\n\s*Function : ", txt)
             if "proj_gemm_kernel" in p.split("\n", 1)[0]]
    assert len(parts) == 3, len(parts)   # STORE, QKV, OUT (3-D A map)
    for p in parts:
        assert p.count("UTCHMMA.2CTA") >= 4
        assert re.search(r"UTMALDG\.[23]D\.2CTA", p)
        assert "LDTM" in p
        assert "LDL" not in p and "STL" not in p


def test_tf32_attention_sass_is_tcgen05():
    """attend_tf32.cu: the f32 attention runs on the tensor cores (UTCHMMA,
    TMA 3-D loads, LDTM / STTM for S, P and O) without spills."""
    if not LIB.exists() or not Path(CUOBJDUMP).exists():
        pytest.skip("library not built or cuobjdump absent")
    txt = subprocess.run([CUOBJDUMP, "-sass", str(LIB)], capture_output=True, text=True,
                         check=True).stdout
    parts = [p for p in re.split(r"\n\s*Function : ", txt)
             if "attend_tf32_kernel" in p.split("\n", 1)[0]]
    assert len(parts) == 1
    p = parts[0]
    assert p.count("UTCHMMA") >= 24 and "UTMALDG.3D" in p
    assert "LDTM" in p and "STTM" in p
    assert "LDL" not in p and "STL" not in p


def test_tf32_pair_attention_sass_is_2cta():
    """The opt-in 2-CTA f32 attention (TSA_TF32_PAIRS=1): paired MMAs
    (UTCHMMA.2CTA) issued by the leader, TMA 3-D loads, no spills."""
    if not LIB.exists() or not Path(CUOBJDUMP).exists():
        pytest.skip("library not built or cuobjdump absent")
    txt = subprocess.run([CUOBJDUMP, "-sass", str(LIB)], capture_output=True, text=True,
                         check=True).stdout
    parts = [p for p in re.split(r"\n\s*Function : ", txt)
             if "attend_tf32_pair_kernel" in p.split("\n", 1)[0]]
    assert len(parts) == 1
    p = parts[0]
    assert p.count("UTCHMMA.2CTA") >= 24 and "UTMALDG.3D" in p
    assert "LDTM" in p and "STTM" in p
    assert "LDL" not in p and "STL" not in p
