"""The C-ABI library loads and exports exactly what include/tw_gemm.h declares
(no compute calls: these run without a GPU)."""

from __future__ import annotations

import ctypes
import re
import subprocess
from pathlib import Path

import pytest

import paper_2402_10876_b200 as tw
from paper_2402_10876_b200 import _build, _native

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "tw_gemm.h"


def declared_functions():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"TW_API\s+[\w\s\*]+?\b(tw_\w+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    _build.build_native()
    return _native.load_library()


def test_header_declares_the_abi():
    names = declared_functions()
    assert "tw_gemm" in names and "tw_plan_create_cto" in names
    assert set(names) == set(_native.SIGNATURES), "ctypes table out of sync with the header"


def test_library_exports_every_declared_symbol(lib):
    for name in declared_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", str(_native.LIB_PATH)],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (tw_\w+)", out))
    assert exported == set(declared_functions())


def test_abi_version(lib):
    assert lib.tw_abi_version() == 421


def test_sass_is_blackwell_native():
    """tcgen05 MMA, TMEM loads, TMA tile loads and TMA stores are in the shipped binary."""
    out = subprocess.run(["cuobjdump", "-sass", str(_native.LIB_PATH)], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    sass = out.stdout
    assert "UTCHMMA" in sass
    assert "UTMALDG.2D" in sass
    assert "UTMASTG.2D" in sass
    assert "LDTM" in sass


def test_status_mapping():
    with pytest.raises(tw.CorruptEncodingError):
        tw.errors.raise_for_status(4, "x")
    with pytest.raises(tw.ContractViolationError):
        tw.errors.raise_for_status(3, "x")
    with pytest.raises(tw.InvalidInputError):
        tw.errors.raise_for_status(2, "x")
    with pytest.raises(tw.DeviceError):
        tw.errors.raise_for_status(5, "x")
    tw.errors.raise_for_status(0, "")


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    rng = __import__("numpy").random.default_rng(0)
    w = rng.normal(size=(8, 8)).astype("float32")
    _, tsm = tw.prune_tw(w, 0.5, 4)
    with pytest.raises(tw.DeviceError):
        tw.gemm_tile_sparse(rng.normal(size=(4, 8)).astype("float32"), tsm)
