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


def test_argument_validation_without_a_device():
    """Every entry point rejects bad arguments with a code and a message before it
    touches the device (these calls run in the CPU container)."""
    import ctypes

    from paper_2404_17344_b200.nufft import NufftPlan

    lib = _native.lib()
    wf = NufftPlan(dims=3, m=32).window_fn()
    out = ctypes.c_void_p()
    q = (ctypes.c_int32 * 1)(3)
    cols = (ctypes.c_int32 * 3)(0, 1, 2)
    X = ctypes.c_void_p(1)  # never dereferenced: validation fails first

    def code(rc, needle):
        assert rc in (_native.AK_ERR_INVALID, _native.AK_ERR_UNSUPPORTED), rc
        assert needle in lib.ak_last_error().decode()

    code(lib.ak_geom_create(64, 1, q, cols, X, 10, 3, ctypes.byref(wf), None, None), "null")
    code(lib.ak_geom_create(1, 1, q, cols, X, 10, 3, ctypes.byref(wf), None, ctypes.byref(out)), "grid size")
    code(lib.ak_geom_create(64, 0, q, cols, X, 10, 3, ctypes.byref(wf), None, ctypes.byref(out)), "window")
    code(lib.ak_geom_create(64, 1, q, cols, None, 10, 3, ctypes.byref(wf), None, ctypes.byref(out)), "point")
    bad_q = (ctypes.c_int32 * 1)(4)
    code(lib.ak_geom_create(64, 1, bad_q, cols, X, 10, 3, ctypes.byref(wf), None, ctypes.byref(out)), "1..3")
    bad_cols = (ctypes.c_int32 * 3)(0, 1, 5)
    code(lib.ak_geom_create(64, 1, q, bad_cols, X, 10, 3, ctypes.byref(wf), None, ctypes.byref(out)), "column")
    wf_bad = NufftPlan(dims=3, m=32).window_fn()
    odd = _native.WindowFn()
    ctypes.memmove(ctypes.byref(odd), ctypes.byref(wf_bad), ctypes.sizeof(odd))
    odd.taps = 11
    code(lib.ak_geom_create(64, 1, q, cols, X, 10, 3, ctypes.byref(odd), None, ctypes.byref(out)), "taps")
    rows_in = (ctypes.c_int64 * 1)(10)
    code(lib.ak_geom_create_masked(64, 1, q, cols, X, 10, 3, None, rows_in, ctypes.byref(wf), None,
                                   ctypes.byref(out)), "null")
    bad_rows = (ctypes.c_int64 * 1)(11)
    code(lib.ak_geom_create_masked(64, 1, q, cols, X, 10, 3, X, bad_rows, ctypes.byref(wf), None,
                                   ctypes.byref(out)), "row count")
    assert out.value is None
    code(lib.ak_spread(None, None, 1, 0, None, None), "spread")
    code(lib.ak_interp(None, None, 1, None, None, 0, 1, 0, None), "interp")
    code(lib.ak_op_create(None, None, 32, 1, 1, None, ctypes.byref(out)), "null")
    code(lib.ak_op_apply(None, None, 0, None, None, None, 0, None, 0, None), "null")
    code(lib.ak_type1_band(4, 64, 32, None, None, None, None, None), "type1")
    code(lib.ak_type2_grid(3, 64, 128, None, None, None, None, None), "type2")
    code(lib.ak_dense_apply(9, 1.0, 1.0, 1, q, cols, None, 0, 3, None, 0, 3, None, None, None, None), "dense")
