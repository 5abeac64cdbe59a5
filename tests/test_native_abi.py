"""The C-ABI library builds for sm_100a, loads, and exports every entry
point include/meshchroma_b200.h declares (no device calls here)."""

import re
import subprocess
from pathlib import Path

import pytest

from paper_1601_07613_b200 import _native

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    text = (ROOT / "include" / "meshchroma_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mc_[a-z0-9_]+)\s*\(", text)))


def test_header_and_binding_agree():
    decl = declared_symbols()
    assert decl, "no declarations parsed"
    assert sorted(_native.EXPORTED) == decl


def test_library_exports_every_symbol():
    lib = _native.lib()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.mc_abi_version() == 1011
    assert lib.mc_device_count() >= 0


def test_library_is_sm100a():
    path = _native.library_path()
    out = subprocess.run(["cuobjdump", "--list-elf", str(path)], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_errors_map_to_reference_types():
    import numpy as np
    import paper_1601_07613_b200 as P
    lib = _native.lib()
    se = np.zeros((0, 2), dtype=np.int64)
    rc = lib.mc_naive_greedy(0, 1, _native.ptr(se), None, None)
    assert rc == _native.MC_EINVAL
    with pytest.raises(ValueError):
        _native.check(rc)
    with pytest.raises(P.WriteConflictError):
        _native.check(_native.MC_ECONFLICT)
