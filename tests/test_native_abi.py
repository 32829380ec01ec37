"""CPU-side checks of the C ABI: the library loads and exports every symbol include/rrg.h declares."""

import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
LIB = ROOT / "paper_2410_18926_b200" / "librrg.so"


def declared_symbols():
    text = (ROOT / "include" / "rrg.h").read_text()
    return sorted(set(re.findall(r"\b(rrg_[a-z_]+)\s*\(", text)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    for s in ["rrg_index_open", "rrg_index_create", "rrg_search", "rrg_search_host", "rrg_last_error"]:
        assert s in syms


def test_library_exports_every_declared_symbol():
    if not LIB.exists():
        subprocess.run(["make", "-C", str(ROOT), "-j4"], check=True)
    out = subprocess.run(["nm", "-D", "--defined-only", str(LIB)], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r" T (rrg_\w+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing


def test_python_binding_loads_and_maps_errors():
    import paper_2410_18926_b200 as pkg
    from paper_2410_18926_b200 import _native

    assert pkg.version().startswith("rrg")
    for name in _native.SIGNATURES:
        assert hasattr(_native.lib, name)
    # a failing call without a GPU still maps to the reference's error taxonomy
    with pytest.raises(pkg.RrannError):
        pkg.DeviceIndex.from_file(ROOT / "does-not-exist.rrr")


def test_format_errors_without_gpu(tmp_path):
    """The native loader parses and CRC-checks before touching the device for malformed files."""
    import numpy as np

    import paper_2410_18926_b200 as pkg
    from conftest import load_golden

    blob = load_golden("euclid_q")["index_bytes"].tobytes()
    p = tmp_path / "bad.rrr"
    p.write_bytes(b"XXXXXXXX" + blob[8:])
    with pytest.raises(pkg.FormatError, match="bad magic"):
        pkg.DeviceIndex.from_file(p)
    del np


def test_errors_subclass_reference(rrann_ref):
    import importlib

    import paper_2410_18926_b200.errors as E
    E = importlib.reload(E)
    assert issubclass(E.ParameterError, rrann_ref.ParameterError)
    assert issubclass(E.ShapeError, rrann_ref.RrannError)
    assert E.DataError.category == "data"


def test_pack_candidates_rejects_int32_offset_overflow():
    """rrg_pack_candidates' offsets are int32: a call whose lists could hold 2^31 entries is
    a ParameterError, raised before any device work (so it runs without a GPU)."""
    import paper_2410_18926_b200 as pkg
    from paper_2410_18926_b200 import _native
    from paper_2410_18926_b200._native import check

    with pytest.raises(pkg.ParameterError, match="int32 offsets"):
        check(_native.lib.rrg_pack_candidates(3_000_000, 800, None, None, None, None, None, None, None))
