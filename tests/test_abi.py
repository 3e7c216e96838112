"""The C-ABI library loads and exports every symbol include/picasso_b200.h declares
(no compute calls — this runs without a GPU)."""

import ctypes
import os
import re

from conftest import ROOT


def _declared():
    with open(os.path.join(ROOT, "include", "picasso_b200.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(pcg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_all_declared_symbols():
    from paper_2401_06713_b200 import _native

    lib = ctypes.CDLL(_native.LIB_PATH)
    names = _declared()
    assert "pcg_count" in names and "pcg_fill" in names
    for name in names:
        assert hasattr(lib, name), name
    assert set(_native.EXPORTED) == set(names)
    assert lib.pcg_version() == 1


def test_library_is_sm100a():
    import subprocess

    from paper_2401_06713_b200 import _native

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _native.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
