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
    code(lib.ak_cg_step(None, 0.1, X, X, X, 10, X, X, 5, X, None), "CG step")
    code(lib.ak_cg_step(X, 0.1, X, X, X, 0, X, X, 5, X, None), "CG step")
    code(lib.ak_cg_step_batched(X, None, 0, X, X, X, X, 10, X, None, 0, X, None), "batched CG")
    code(lib.ak_cg_step_batched(X, None, 2, None, X, X, X, 10, X, None, 0, X, None), "batched CG")


def test_tuning_defaults_and_validation():
    """ak_tuning: the defaults the library uses (the measured heuristics)
    and rejection of out-of-range values by ak_geom_create_ex before any device work.
    The library reads no environment variables (the kernel choice is a plan property)."""
    import ctypes

    import pytest

    from paper_2404_17344_b200.nufft import NufftPlan

    t = _native.tuning()
    assert (t.weight_tables, t.cell_items3, t.cell_items2, t.chunk3, t.rhs_pair_spread, t.fused_fft3,
            t.generic_kernels, t.sparse_warps, t.tc_spread3) == (1, 0, 0, 0, 1, 1, 0, 2, 3)
    assert (t.dense_cells3, t.dense_cells3_interp, t.dense_cells2) == (300.0, 64.0, 2.0)
    with pytest.raises(ValueError):
        _native.tuning(no_such_knob=1)
    lib = _native.lib()
    wf = NufftPlan(dims=3, m=32).window_fn()
    out = ctypes.c_void_p()
    q = (ctypes.c_int32 * 1)(3)
    cols = (ctypes.c_int32 * 3)(0, 1, 2)
    X = ctypes.c_void_p(1)
    for bad in ({"cell_items3": 3}, {"cell_items2": 2}, {"chunk3": 10}, {"dense_cells3": -1.0}, {"sparse_warps": 3},
                {"tc_spread3": 4}):
        rc = lib.ak_geom_create_ex(64, 1, q, cols, X, 10, 3, None, None, ctypes.byref(wf),
                                   ctypes.byref(_native.tuning(**bad)), None, ctypes.byref(out))
        assert rc == _native.AK_ERR_INVALID and b"tuning" in lib.ak_last_error(), bad
    rows_in = (ctypes.c_int64 * 1)(10)
    rc = lib.ak_geom_create_ex(64, 1, q, cols, X, 10, 3, None, rows_in, ctypes.byref(wf), None, None,
                               ctypes.byref(out))
    assert rc == _native.AK_ERR_INVALID
    # no environment reads in the library's own sources (the CUDA runtime linked into it
    # reads CUDA_* variables itself)
    for src in (ROOT / "paper_2404_17344_b200" / "csrc").iterdir():
        assert "getenv" not in src.read_text(), src.name


def test_profiler_report_empty_without_launches():
    lib = _native.lib()
    assert lib.ak_prof_enable(0) == 0
    assert lib.ak_prof_reset() == 0
    assert lib.ak_prof_report(None, 0) == 1   # empty report: just the terminator
