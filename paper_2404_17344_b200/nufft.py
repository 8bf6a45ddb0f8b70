"""Nonuniform FFTs on [-1/2, 1/2)^q, q in {1, 2, 3}, on the B200.

API parity with ``addkern.nufft`` (/root/reference/pkg/src/addkern/nufft.py):

    type-1   S_k    = sum_j v_j exp(-2 pi i k.x_j)      (nufft_type1, :346-365)
    type-2   f(x_j) = sum_k c_k exp(+2 pi i k.x_j)      (nufft_type2, :368-394)

with the same oversampled grid n = 2*ceil(sigma*m/2), the same Kaiser-Bessel
(Beatty shape parameter) or Gaussian window with 2*cutoff taps per axis, the
same FFT frequency ordering and the same deconvolution (-1)^k / psi_hat(k/n).

What differs is where the work runs: ``prepare_points`` bin-sorts the points
on the GPU (libaddkern_b200: ak_geom_create) instead of tabulating per-point
window weights, and the window weights are evaluated inside the spread /
interp kernels from a per-tap polynomial fit of the window (``window_fn``),
accurate to ~1e-14 of the window peak.  Plan constants (n, beta, psi_hat,
deconvolution) are computed on the host exactly as the reference does.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .errors import PointOutOfDomainError

KAISER_BESSEL = "kaiser_bessel"
GAUSSIAN_WINDOW = "gaussian_window"

#: polynomial degree of the per-tap window fit (AK_NCOEF even + AK_NCOEF odd coefficients)
WINDOW_POLY_DEGREE = 2 * _native.AK_NCOEF - 1
#: the fit is rejected if it is worse than this (absolute, window peak = 1).  Cutoffs
#: below 4 have NUFFT errors >= 1e-5 of their own, so their fit may be coarser.
WINDOW_FIT_TOL = 5e-13
WINDOW_FIT_TOL_SMALL_CUTOFF = 1e-10


def freqs(m: int) -> np.ndarray:
    """Integer frequencies of I_m in FFT order: 0..m/2-1, -m/2..-1 (nufft.py:38-40)."""
    return (np.fft.fftfreq(m) * m).astype(np.int64)


def grid_positions(m: int) -> np.ndarray:
    """Sampling positions j/m in FFT order (nufft.py:43-45)."""
    return np.fft.fftfreq(m)


@dataclass(frozen=True)
class CoefficientTable:
    """Fourier coefficients c_k on the tensor grid I_m, FFT ordering (nufft.py:48-62)."""

    dims: int
    m: int
    values: np.ndarray

    def __post_init__(self):
        vals = np.asarray(self.values, dtype=np.complex128)
        object.__setattr__(self, "values", vals)
        if vals.shape != (self.m,) * self.dims:
            raise ValueError(f"expected shape {(self.m,) * self.dims}, got {vals.shape}")
        if not np.all(np.isfinite(vals.real)) or not np.all(np.isfinite(vals.imag)):
            raise ValueError("coefficients must be finite")


def grid_fft_coefficients(samples) -> CoefficientTable:
    """c_k = m^-q sum_j f(j/m) exp(-2 pi i j.k/m) (nufft.py:65-77); plan-time, tiny."""
    samples = np.asarray(samples)
    m = samples.shape[0]
    if samples.shape != (m,) * samples.ndim or m % 2:
        raise ValueError("samples must form an even cubic grid")
    return CoefficientTable(dims=samples.ndim, m=m, values=np.fft.fftn(samples) / samples.size)


def coefficients_to_samples(table: CoefficientTable) -> np.ndarray:
    """Inverse of grid_fft_coefficients (nufft.py:80-82)."""
    return np.fft.ifftn(table.values) * table.values.size


@dataclass(frozen=True)
class NufftPlan:
    """Transform sizes and window configuration (nufft.py:85-157)."""

    dims: int
    m: int
    oversampling: float = 2.0
    cutoff: int = 6
    window: str = KAISER_BESSEL
    n: int = field(init=False)
    beta: float = field(init=False)

    def __post_init__(self):
        if self.dims not in (1, 2, 3):
            raise ValueError("dims must be 1, 2 or 3")
        if self.m < 2 or self.m % 2:
            raise ValueError("m must be even and >= 2")
        if self.oversampling < 1.25:
            raise ValueError("oversampling must be >= 1.25")
        if self.cutoff < 2:
            raise ValueError("cutoff must be >= 2")
        if self.window not in (KAISER_BESSEL, GAUSSIAN_WINDOW):
            raise ValueError(f"unknown window {self.window!r}")
        if 2 * self.cutoff > _native.AK_MAX_TAPS:
            raise ValueError(f"cutoff must be <= {_native.AK_MAX_TAPS // 2} on the GPU path")
        n = 2 * int(math.ceil(self.oversampling * self.m / 2.0))
        sigma = n / self.m
        taps = 2 * self.cutoff
        if self.window == KAISER_BESSEL:
            # Beatty et al. shape parameter for the realised oversampling (nufft.py:112-115)
            beta = math.pi * math.sqrt((taps / sigma) ** 2 * (sigma - 0.5) ** 2 - 0.8)
        else:
            beta = 2.0 * sigma * self.cutoff / ((2.0 * sigma - 1.0) * math.pi)
        object.__setattr__(self, "n", n)
        object.__setattr__(self, "beta", beta)

    @property
    def taps(self) -> int:
        return 2 * self.cutoff

    def window_values(self, z) -> np.ndarray:
        """Window at offsets z (grid cells), peak 1 (nufft.py:125-131)."""
        z = np.asarray(z, dtype=np.float64)
        if self.window == KAISER_BESSEL:
            arg = np.maximum(0.0, 1.0 - (z / self.cutoff) ** 2)
            return np.i0(self.beta * np.sqrt(arg)) / np.i0(self.beta)
        return np.exp(-(z * z) / self.beta)

    def window_transform(self, k) -> np.ndarray:
        """Continuous Fourier transform of the window at k/n (nufft.py:133-147)."""
        nu = np.asarray(k, dtype=np.float64) / self.n
        c = float(self.cutoff)
        if self.window == KAISER_BESSEL:
            arg = self.beta ** 2 - (2.0 * math.pi * c * nu) ** 2
            root = np.sqrt(np.maximum(arg, 1e-300))
            out = 2.0 * c * np.sinh(root) / (root * np.i0(self.beta))
            osc = arg < 0
            if np.any(osc):
                ro = np.sqrt(-arg[osc])
                out[osc] = 2.0 * c * np.sin(ro) / (ro * np.i0(self.beta))
            return out
        return np.sqrt(math.pi * self.beta) * np.exp(-((math.pi * nu) ** 2) * self.beta)

    def deconvolution(self) -> np.ndarray:
        """(-1)^k / psi_hat(k/n) per axis, FFT order (nufft.py:149-157)."""
        k = freqs(self.m)
        return (1.0 - 2.0 * (k & 1)) / self.window_transform(k)

    def band_deconvolution_squared(self) -> np.ndarray:
        """1 / psi_hat(k/n)^2: both deconvolutions of a type-1 -> type-2 round trip."""
        return 1.0 / self.window_transform(freqs(self.m)) ** 2

    def window_fn(self) -> "_native.WindowFn":
        """Per-tap polynomial table of the window for the CUDA kernels (cached).

        Tap counts without specialised kernels are padded with one zero tap on
        each side (the window is zero there: identical sums): 6 -> 8 and
        10 -> 12 taps, so cutoffs 3 and 5 run on the tuned 8- and 12-tap kernels
        (12: tensor-core interpolation, plan-time weight tables) instead of the
        one-thread-per-point fallback.
        """
        cached = _WINDOW_CACHE.get(self._wkey())
        if cached is None:
            cached = _fit_window(self)
            if cached.taps in PADDED_TAPS:
                cached = _pad_window(cached, PADDED_TAPS[cached.taps])
            _WINDOW_CACHE[self._wkey()] = cached
        return cached

    def _wkey(self):
        return (self.n, self.cutoff, self.window, self.beta)


_WINDOW_CACHE: dict = {}

#: kernel tap count used for window tap counts that have no specialised kernels
PADDED_TAPS = {6: 8, 10: 12}


def _pad_window(wf: "_native.WindowFn", taps: int) -> "_native.WindowFn":
    """The same window on `taps` >= wf.taps kernel taps: (taps - wf.taps) / 2 zero taps on
    each side.  Pair a of the padded table (taps a and taps-1-a) is pair a - k of the
    original, k = (taps - wf.taps) / 2; the outer k pairs are zero."""
    k = (taps - wf.taps) // 2
    out = _native.WindowFn()
    out.taps = taps
    out.ncoef = wf.ncoef
    for a in range(taps // 2):
        for j in range(_native.AK_NCOEF):
            out.ce[a][j] = wf.ce[a - k][j] if a >= k else 0.0
            out.co[a][j] = wf.co[a - k][j] if a >= k else 0.0
    return out


def _fit_window(plan: NufftPlan) -> "_native.WindowFn":
    """Chebyshev fit of phi(frac + c-1-a) in s = 2 frac - 1, one polynomial per tap.

    Taps a and T-1-a are mirror images (phi is even), so only T/2 fits are
    stored as even/odd parts: w_a = E_a(s^2) + s O_a(s^2),
    w_{T-1-a} = E_a(s^2) - s O_a(s^2).
    """
    from numpy.polynomial import chebyshev as cheb

    T, c, deg = plan.taps, plan.cutoff, WINDOW_POLY_DEGREE
    wf = _native.WindowFn()
    wf.taps = T
    wf.ncoef = _native.AK_NCOEF
    probe = np.linspace(-1.0, 1.0, 2049)
    worst = 0.0
    for a in range(T // 2):
        def g(s, a=a):
            return plan.window_values((s + 1.0) * 0.5 + (c - 1 - a))

        coef = cheb.cheb2poly(cheb.chebinterpolate(g, deg))
        coef = np.concatenate([coef, np.zeros(deg + 1 - coef.size)])
        even, odd = coef[0::2], coef[1::2]
        for k in range(_native.AK_NCOEF):
            wf.ce[a][k] = even[_native.AK_NCOEF - 1 - k]
            wf.co[a][k] = odd[_native.AK_NCOEF - 1 - k]
        s2 = probe * probe
        e = np.polyval(even[::-1], s2)
        o = np.polyval(odd[::-1], s2)
        worst = max(worst, np.max(np.abs(e + probe * o - g(probe))),
                    np.max(np.abs(e - probe * o - g(-probe))))
    tol = WINDOW_FIT_TOL if c >= 4 else WINDOW_FIT_TOL_SMALL_CUTOFF
    if worst > tol:
        raise ValueError(f"window polynomial fit error {worst:.2e} exceeds {tol:.0e}")
    return wf


# ---------------------------------------------------------------------------
# device geometry


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise _native.NativeLibraryError("a CUDA device is required: the fast summation has no CPU path")
    return torch


def _stream_ptr(torch):
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


class DeviceGeometry:
    """Bin-sorted nodes of P windows on the device (replaces the per-window
    ``SpreadGeometry`` tuple, nufft.py:160-191).  Immutable; owns device memory."""

    def __init__(self, n: int, qs, cols, features, window_fn, row_masks=None, tuning=None):
        """row_masks: optional (P, N) bool array -- window w uses only the rows with
        row_masks[w] set (the multi-GPU cell-slab layout).  tuning: optional dict of
        ak_tuning fields that pin the plan's kernel choices (tests; the defaults are
        the library's measured heuristics) -- ak_geom_create_ex."""
        torch = _torch()
        lib = _native.lib()
        feats = features
        if not (isinstance(feats, torch.Tensor) and feats.is_cuda):
            feats = torch.as_tensor(np.ascontiguousarray(features, dtype=np.float64), device="cuda")
        feats = feats.to(torch.float64).contiguous()
        if feats.ndim != 2:
            raise ValueError("features must be 2-D")
        P = len(qs)
        qarr = (ctypes.c_int32 * P)(*[int(q) for q in qs])
        flat = []
        for q, cs in zip(qs, cols):
            cs = list(cs)
            if len(cs) != q:
                raise ValueError("window columns do not match its length")
            flat.extend(cs + [0] * (3 - q))
        carr = (ctypes.c_int32 * (3 * P))(*flat)
        self._lib = lib
        self._handle = ctypes.c_void_p()
        self.n = int(n)
        self.qs = tuple(int(q) for q in qs)
        self.cols = tuple(tuple(int(c) for c in cs) for cs in cols)
        self.n_points = int(feats.shape[0])
        self.rows_per_window = (self.n_points,) * P
        md, rows_in = None, None
        if row_masks is not None:
            m = np.ascontiguousarray(np.asarray(row_masks, dtype=bool))
            if m.shape != (P, self.n_points):
                raise ValueError("row_masks must have shape (windows, rows)")
            md = torch.as_tensor(m.view(np.uint8), device="cuda")
            self.rows_per_window = tuple(int(c) for c in m.sum(axis=1))
            rows_in = (ctypes.c_int64 * P)(*self.rows_per_window)
        tune = _native.tuning(**(tuning or {}))
        rc = lib.ak_geom_create_ex(self.n, P, qarr, carr, ctypes.c_void_p(feats.data_ptr()), self.n_points,
                                   int(feats.shape[1]), ctypes.c_void_p(md.data_ptr() if md is not None else 0),
                                   rows_in, ctypes.byref(window_fn), ctypes.byref(tune), _stream_ptr(torch),
                                   ctypes.byref(self._handle))
        _native.check(rc, "ak_geom_create_ex")
        self.describe = (lib.ak_geom_describe(self._handle) or b"").decode()
        self.tuning = dict(tuning) if tuning else None
        self.n_windows = P
        self.n_items = int(lib.ak_geom_num_items(self._handle))
        self.canon_total = int(lib.ak_geom_canon_total(self._handle))
        self.canon_offsets = tuple(int(lib.ak_geom_canon_offset(self._handle, w)) for w in range(P))
        self.boxes = tuple(self._box(lib, w) for w in range(P))

    def _box(self, lib, w: int):
        """((lo, L) per axis): window w's occupied grid box (ak_geom_box)."""
        b = (ctypes.c_int32 * 6)()
        _native.check(lib.ak_geom_box(self._handle, w, b), "ak_geom_box")
        return tuple((int(b[2 * a]), int(b[2 * a + 1])) for a in range(3))

    @property
    def handle(self) -> ctypes.c_void_p:
        return self._handle

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None and h.value:
            try:
                self._lib.ak_geom_destroy(h)
            except Exception:  # pragma: no cover - interpreter shutdown
                pass
            self._handle = None


# Backwards-compatible name: one window's device geometry.
SpreadGeometry = DeviceGeometry


def _points_array(plan: NufftPlan, points) -> np.ndarray:
    pts = np.atleast_2d(np.asarray(points, dtype=np.float64))
    if plan.dims == 1 and pts.shape[0] == 1 and pts.shape[1] != 1:
        pts = pts.T
    if pts.ndim != 2 or pts.shape[1] != plan.dims:
        raise ValueError(f"points must have shape (N, {plan.dims})")
    return np.ascontiguousarray(pts)


def prepare_points(plan: NufftPlan, points, tuning=None) -> DeviceGeometry:
    """Validate nodes and bin-sort them on the GPU (nufft.py:169-191).  ``tuning``
    (extension): ak_tuning fields pinning the kernel choices (DeviceGeometry)."""
    pts = _points_array(plan, points)
    if np.any(pts < -0.5) or np.any(pts >= 0.5):
        raise PointOutOfDomainError("points must lie in [-1/2, 1/2)")
    return DeviceGeometry(plan.n, (plan.dims,), (tuple(range(plan.dims)),), pts, plan.window_fn(), tuning=tuning)


def _as_geometry(plan: NufftPlan, points) -> DeviceGeometry:
    if isinstance(points, DeviceGeometry):
        if points.n_windows != 1 or points.qs[0] != plan.dims or points.n != plan.n:
            raise ValueError("geometry does not match the plan")
        return points
    return prepare_points(plan, points)


def _deconv_device(plan: NufftPlan, torch):
    d = plan.deconvolution()
    return torch.as_tensor(np.tile(d, 3), dtype=torch.float64, device="cuda")


def nufft_type1(plan: NufftPlan, points, weights) -> np.ndarray:
    """S_k = sum_j v_j e^{-2 pi i k.x_j}, k in I_m, FFT order (nufft.py:346-365)."""
    torch = _torch()
    lib = _native.lib()
    geom = _as_geometry(plan, points)
    w = np.asarray(weights, dtype=np.complex128)
    if w.shape != (geom.n_points,):
        raise ValueError("weights length must match the number of points")
    N = geom.n_points
    V = torch.as_tensor(np.stack([w.real, w.imag]), dtype=torch.float64, device="cuda").contiguous()
    ng = plan.n ** plan.dims
    grids = torch.zeros(2 * ng, dtype=torch.float64, device="cuda")
    st = _stream_ptr(torch)
    if N:
        _native.check(lib.ak_spread(geom.handle, V.data_ptr(), 2, N, grids.data_ptr(), st), "ak_spread")
    S = torch.empty(2 * plan.m ** plan.dims, dtype=torch.float64, device="cuda")
    dec = _deconv_device(plan, torch)
    _native.check(lib.ak_type1_band(plan.dims, plan.n, plan.m, grids.data_ptr(), grids.data_ptr() + 8 * ng,
                                    dec.data_ptr(), S.data_ptr(), st), "ak_type1_band")
    out = S.cpu().numpy().view(np.complex128)
    return out.reshape((plan.m,) * plan.dims)


def nufft_type2(plan: NufftPlan, points, coeffs) -> np.ndarray:
    """f(x_j) = sum_k c_k e^{+2 pi i k.x_j} at the nodes (nufft.py:368-394)."""
    torch = _torch()
    lib = _native.lib()
    geom = _as_geometry(plan, points)
    if isinstance(coeffs, CoefficientTable):
        if coeffs.dims != plan.dims or coeffs.m != plan.m:
            raise ValueError("coefficient table does not match the plan")
        vals = coeffs.values
    else:
        vals = np.asarray(coeffs, dtype=np.complex128)
        if vals.shape != (plan.m,) * plan.dims:
            raise ValueError(f"coefficients must have shape {(plan.m,) * plan.dims}")
    N = geom.n_points
    c = torch.as_tensor(np.ascontiguousarray(vals).view(np.float64).ravel(), device="cuda")
    ng = plan.n ** plan.dims
    grids = torch.empty(2 * ng, dtype=torch.float64, device="cuda")
    dec = _deconv_device(plan, torch)
    st = _stream_ptr(torch)
    _native.check(lib.ak_type2_grid(plan.dims, plan.n, plan.m, c.data_ptr(), dec.data_ptr(), grids.data_ptr(),
                                    grids.data_ptr() + 8 * ng, st), "ak_type2_grid")
    out = torch.zeros((2, max(N, 1)), dtype=torch.float64, device="cuda")
    one = torch.ones(1, dtype=torch.float64, device="cuda")
    if N:
        _native.check(lib.ak_interp(geom.handle, grids.data_ptr(), 2, one.data_ptr(), out.data_ptr(), out.shape[1],
                                    1, 0, st), "ak_interp")
    o = out.cpu().numpy()[:, :N]
    return o[0] + 1j * o[1]
