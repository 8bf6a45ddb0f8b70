"""ctypes binding of libaddkern_b200.so (the C ABI in include/addkern_b200.h).

There is no CPU fallback: if the library is missing or cannot be loaded the
import of the compute modules fails loudly with ``NativeLibraryError``.
Device memory, streams and pointers come from torch CUDA tensors.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .errors import NativeLibraryError, PointOutOfDomainError

_PKG = Path(__file__).resolve().parent
# AK_LIB_PATH: load a variant build instead (tuning experiments, tools/build_variant.py)
LIB_PATH = Path(os.environ["AK_LIB_PATH"]) if os.environ.get("AK_LIB_PATH") else _PKG / "libaddkern_b200.so"

AK_OK = 0
AK_ERR_INVALID = -1
AK_ERR_CUDA = -2
AK_ERR_DOMAIN = -3
AK_ERR_ALLOC = -4
AK_ERR_CUFFT = -5
AK_ERR_UNSUPPORTED = -6

AK_APPLY_ACCUMULATE = 1
AK_APPLY_SPREAD_ONLY = 2
AK_APPLY_FROM_GRIDS = 4
AK_APPLY_H_PER_RHS = 8
AK_APPLY_SPECTRUM_ONLY = 16
AK_APPLY_FROM_SPECTRUM = 32
AK_APPLY_RHS_MINOR = 64

AK_MAX_TAPS = 16
AK_MAX_PAIRS = 8
AK_NCOEF = 7

#: symbols the header declares; tests check the library exports every one
EXPORTED = (
    "ak_last_error", "ak_version", "ak_launch_count",
    "ak_geom_create", "ak_geom_create_masked", "ak_geom_destroy", "ak_geom_num_points", "ak_geom_num_windows",
    "ak_geom_num_items", "ak_geom_grid_elems", "ak_geom_canon_offset", "ak_geom_canon_total",
    "ak_spread", "ak_interp", "ak_op_create", "ak_op_destroy", "ak_op_apply", "ak_op_grids", "ak_op_band",
    "ak_type1_band", "ak_type2_grid", "ak_dense_apply", "ak_probe_fp64", "ak_probe_dmma",
    "ak_tuning_default", "ak_geom_create_ex", "ak_geom_describe", "ak_prof_enable", "ak_prof_reset",
    "ak_prof_report", "ak_geom_box", "ak_cg_step", "ak_cg_step_batched",
)

# ak_cg_step state layout (include/addkern_b200.h)
AK_CG_RS, AK_CG_ACTIVE, AK_CG_ITERATIONS, AK_CG_BREAKDOWN_AT, AK_CG_BREAKDOWN_PAP, AK_CG_THRESHOLD = range(6)
AK_CG_STATE = 8
AK_CG_WORK = 2048

FAMILY_CODE = {"gauss": 0, "der_gauss": 1, "matern12": 2, "der_matern12": 3}


class WindowFn(ctypes.Structure):
    _fields_ = [
        ("taps", ctypes.c_int32),
        ("ncoef", ctypes.c_int32),
        ("ce", (ctypes.c_double * AK_NCOEF) * AK_MAX_PAIRS),
        ("co", (ctypes.c_double * AK_NCOEF) * AK_MAX_PAIRS),
    ]


class Tuning(ctypes.Structure):
    """ak_tuning (include/addkern_b200.h): plan-time kernel selection."""

    _fields_ = [
        ("weight_tables", ctypes.c_int32),
        ("cell_items3", ctypes.c_int32),
        ("dense_cells3", ctypes.c_double),
        ("dense_cells3_interp", ctypes.c_double),
        ("cell_items2", ctypes.c_int32),
        ("dense_cells2", ctypes.c_double),
        ("chunk3", ctypes.c_int32),
        ("rhs_pair_spread", ctypes.c_int32),
        ("fused_fft3", ctypes.c_int32),
        ("generic_kernels", ctypes.c_int32),
        ("sparse_warps", ctypes.c_int32),
        ("tc_spread3", ctypes.c_int32),
    ]


def tuning(**overrides) -> Tuning:
    """The library's default tuning with the given fields replaced (unknown names raise)."""
    t = Tuning()
    lib().ak_tuning_default(ctypes.byref(t))
    names = {f[0] for f in Tuning._fields_}
    for k, v in overrides.items():
        if k not in names:
            raise ValueError(f"unknown tuning field {k!r}")
        setattr(t, k, v)
    return t


_c_int = ctypes.c_int
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_vp = ctypes.c_void_p
_dp = ctypes.c_void_p  # device pointers travel as integers


def _declare(lib: ctypes.CDLL) -> None:
    sig = {
        "ak_last_error": (ctypes.c_char_p, []),
        "ak_version": (ctypes.c_char_p, []),
        "ak_launch_count": (_i64, []),
        "ak_geom_create": (_c_int, [_i32, _i32, ctypes.POINTER(_i32), ctypes.POINTER(_i32), _dp, _i64, _i64,
                                    ctypes.POINTER(WindowFn), _vp, ctypes.POINTER(_vp)]),
        "ak_geom_create_masked": (_c_int, [_i32, _i32, ctypes.POINTER(_i32), ctypes.POINTER(_i32), _dp, _i64, _i64,
                                           _dp, ctypes.POINTER(_i64), ctypes.POINTER(WindowFn), _vp,
                                           ctypes.POINTER(_vp)]),
        "ak_geom_create_ex": (_c_int, [_i32, _i32, ctypes.POINTER(_i32), ctypes.POINTER(_i32), _dp, _i64, _i64,
                                       _dp, ctypes.POINTER(_i64), ctypes.POINTER(WindowFn), ctypes.POINTER(Tuning),
                                       _vp, ctypes.POINTER(_vp)]),
        "ak_tuning_default": (None, [ctypes.POINTER(Tuning)]),
        "ak_geom_describe": (ctypes.c_char_p, [_vp]),
        "ak_prof_enable": (_c_int, [_i32]),
        "ak_prof_reset": (_c_int, []),
        "ak_prof_report": (_i64, [ctypes.c_char_p, _i64]),
        "ak_geom_destroy": (_c_int, [_vp]),
        "ak_geom_num_points": (_i64, [_vp]),
        "ak_geom_num_windows": (_i32, [_vp]),
        "ak_geom_num_items": (_i64, [_vp]),
        "ak_geom_grid_elems": (_i64, [_vp, _i32]),
        "ak_geom_canon_offset": (_i64, [_vp, _i32]),
        "ak_geom_canon_total": (_i64, [_vp]),
        "ak_geom_box": (_c_int, [_vp, _i32, ctypes.POINTER(_i32)]),
        "ak_spread": (_c_int, [_vp, _dp, _i32, _i64, _dp, _vp]),
        "ak_interp": (_c_int, [_vp, _dp, _i32, _dp, _dp, _i64, _i32, _i64, _vp]),
        "ak_op_create": (_c_int, [_vp, _vp, _i32, _i32, _i32, _vp, ctypes.POINTER(_vp)]),
        "ak_op_destroy": (_c_int, [_vp]),
        "ak_op_grids": (_c_int, [_vp, ctypes.POINTER(_vp), ctypes.POINTER(_i64)]),
        "ak_op_band": (_c_int, [_vp, ctypes.POINTER(_vp), ctypes.POINTER(_i64)]),
        "ak_op_apply": (_c_int, [_vp, _dp, _i64, _dp, _dp, ctypes.POINTER(_vp), _i64, ctypes.POINTER(_i32),
                                 _i32, _vp]),
        "ak_type1_band": (_c_int, [_i32, _i32, _i32, _dp, _dp, _dp, _dp, _vp]),
        "ak_type2_grid": (_c_int, [_i32, _i32, _i32, _dp, _dp, _dp, _dp, _vp]),
        "ak_dense_apply": (_c_int, [_i32, ctypes.c_double, ctypes.c_double, _i32, ctypes.POINTER(_i32),
                                    ctypes.POINTER(_i32), _dp, _i64, _i64, _dp, _i64, _i64, _dp, _dp, _dp, _vp]),
        "ak_cg_step": (_c_int, [_dp, ctypes.c_double, _dp, _dp, _dp, _i64, _dp, _dp, _i64, _dp, _vp]),
        "ak_cg_step_batched": (_c_int, [_dp, _dp, _i32, _dp, _dp, _dp, _dp, _i64, _dp, _dp, _i64, _dp, _vp]),
        "ak_probe_fp64": (_c_int, [_i64, _vp, ctypes.POINTER(ctypes.c_double)]),
        "ak_probe_dmma": (_c_int, [_i64, _vp, ctypes.POINTER(ctypes.c_double)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args


_LIB = None


def lib() -> ctypes.CDLL:
    """Load (once) and return the native library; raises if it is unavailable."""
    global _LIB
    if _LIB is None:
        if not LIB_PATH.exists():
            if os.environ.get("AK_AUTOBUILD", "1") == "1":
                from .build import build
                build()
            if not LIB_PATH.exists():
                raise NativeLibraryError(f"{LIB_PATH} is missing; run `python -m paper_2404_17344_b200.build`")
        try:
            handle = ctypes.CDLL(str(LIB_PATH))
        except OSError as exc:  # pragma: no cover - environment dependent
            raise NativeLibraryError(f"cannot load {LIB_PATH}: {exc}") from exc
        _declare(handle)
        _LIB = handle
    return _LIB


def last_error() -> str:
    msg = lib().ak_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str = "") -> None:
    """Map a C-ABI return code onto the package's exception types."""
    if rc == AK_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if rc == AK_ERR_DOMAIN:
        raise PointOutOfDomainError(msg)
    if rc in (AK_ERR_INVALID, AK_ERR_UNSUPPORTED):
        raise ValueError(msg)
    if rc == AK_ERR_ALLOC:
        raise MemoryError(msg)
    raise NativeLibraryError(msg)


def launch_count() -> int:
    return int(lib().ak_launch_count())


class KernelTimer:
    """Per-kernel device time of everything the library launches inside the block
    (ak_prof_*: CUDA events around each launch on its stream).  Diagnostics only:
    the events add a little overhead, so timed benchmark regions run without it.

        with KernelTimer() as kt:
            fast_matvecs(plan, V)
        kt.report  ->  {"k_spread3c": (launches, total_ms), ...}
    """

    def __enter__(self):
        L = lib()
        L.ak_prof_reset()
        L.ak_prof_enable(1)
        self.report = {}
        return self

    def __exit__(self, *exc):
        L = lib()
        L.ak_prof_enable(0)
        need = int(L.ak_prof_report(None, 0))
        buf = ctypes.create_string_buffer(max(need, 1))
        L.ak_prof_report(buf, need)
        L.ak_prof_reset()
        for line in buf.value.decode().splitlines():
            name, cnt, ms = line.split("\t")
            self.report[name] = (int(cnt), float(ms))
        return False
