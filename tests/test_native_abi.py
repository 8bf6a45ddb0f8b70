"""The C-ABI library builds, loads, and exports every symbol the header
declares (no compute calls: CPU container)."""

import re

from conftest import ROOT
from paper_2404_17344_b200 import _native


def header_functions():
    text = (ROOT / "include" / "addkern_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ak_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_binding_table():
    assert set(header_functions()) == set(_native.EXPORTED)


def test_library_exports_every_declared_symbol():
    lib = _native.lib()
    for name in header_functions():
        assert hasattr(lib, name), name


def test_version_and_counters():
    lib = _native.lib()
    assert b"sm_100a" in lib.ak_version()
    assert _native.launch_count() >= 0


def test_error_mapping():
    import pytest

    from paper_2404_17344_b200.errors import NativeLibraryError, PointOutOfDomainError

    with pytest.raises(PointOutOfDomainError):
        _native.check(_native.AK_ERR_DOMAIN)
    with pytest.raises(ValueError):
        _native.check(_native.AK_ERR_INVALID)
    with pytest.raises(MemoryError):
        _native.check(_native.AK_ERR_ALLOC)
    with pytest.raises(NativeLibraryError):
        _native.check(_native.AK_ERR_CUDA)
    _native.check(_native.AK_OK)


def test_sm100a_cubin_present():
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_native.LIB_PATH)],
                         capture_output=True, text=True)
    assert "sm_100a" in out.stdout
