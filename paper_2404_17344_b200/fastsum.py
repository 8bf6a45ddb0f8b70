"""NFFT fast summation for the additive kernel and its derivatives, on the B200.

Per window s the reference approximates K_s v as

    type-1 NUFFT of v  ->  multiply by the kernel's Fourier coefficients  ->  type-2 NUFFT

summed over windows and scaled by sigma_f^2 (times 2/ell or 1/ell for the
derivative families): /root/reference/pkg/src/addkern/fastsum.py:150-160.

This module keeps that API (build_plan, fast_matvec, fast_dsigma_matvec,
prepare_eval_points, fast_cross_matvec, kernel_coefficients, resolve_m,
PRESETS, AccuracyWarning) and runs the product as one stream-ordered GPU
pipeline per call (libaddkern_b200, ak_op_apply):

    bin-sorted real spread of every (window, RHS)            [CUDA, FP64]
    -> band of the forward transform                          [3-D: band-pruned DFT GEMMs
                                                               on the FP64 tensor cores;
                                                               1-/2-D: batched cuFFT D2Z]
    -> multiply by H = Re(c_hat) / psi_hat^2 per coefficient set (fused into the
       3-D inverse; a band-multiply kernel otherwise)
    -> inverse transform of the band                          [3-D fused / cuFFT Z2D]
    -> interpolation, scaled and summed over windows          [CUDA, FP64]

For real v the reference's complex pipeline has an imaginary part that is
zero up to rounding (its 1e-8 check, fastsum.py:141-147, never fires), so the
real pipeline computes the same numbers.  One spread serves several
coefficient sets, so K v and dK/d ell v (``fast_matvecs``) cost one spread,
one forward FFT, two multiplies, two inverse FFTs and two interps; the
reference needs a separate der_* plan and repeats everything.

Inputs may be numpy arrays (copied to and from the device inside the call,
like the reference's own numpy interface) or torch CUDA tensors (kept on the
device; the product is returned as a CUDA tensor).
"""

from __future__ import annotations

import ctypes
import math
import warnings
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .dataset import PRESCALED, Dataset, same_scaling
from .errors import InvalidScalingError, ScalingMismatchError
from .kernels import DERIVATIVE_FAMILY, DERIVATIVE_PREFACTOR, KernelSpec, radial_profile
from .nufft import (CoefficientTable, DeviceGeometry, NufftPlan, _stream_ptr, _torch,
                    grid_fft_coefficients, grid_positions)
from .windows import WindowSet

PRESETS = {"fine": 64, "default": 32, "rough": 16}


class AccuracyWarning(UserWarning):
    """eta = ell*pi*m/sqrt(2) < 1: the Fourier error may exceed 10 (fastsum.py:39-40)."""


def resolve_m(preset) -> int:
    """fine/default/rough -> 64/32/16, or an explicit even m >= 2 (fastsum.py:43-52)."""
    if isinstance(preset, str):
        if preset not in PRESETS:
            raise ValueError(f"unknown preset {preset!r}; use fine/default/rough")
        return PRESETS[preset]
    m = int(preset)
    if m < 2 or m % 2:
        raise ValueError("explicit m must be even and >= 2")
    return m


def kernel_coefficients(family: str, ell: float, q: int, m: int,
                        symmetric_band: bool = True) -> CoefficientTable:
    """FFT coefficients of the radial kernel sampled on the full m^q grid.

    Simple periodic continuation over [-1/2, 1/2)^q; with ``symmetric_band``
    the unpaired k = -m/2 hyperplanes are zeroed so the trigonometric
    polynomial is real and even (fastsum.py:55-76).  Plan-time, host.
    """
    axis = grid_positions(m)
    r2 = np.zeros((m,) * q)
    for a in range(q):
        shape = [1] * q
        shape[a] = m
        r2 = r2 + (axis * axis).reshape(shape)
    table = grid_fft_coefficients(radial_profile(family, ell, r2))
    if not symmetric_band:
        return table
    vals = table.values.copy()
    for a in range(q):
        idx = [slice(None)] * q
        idx[a] = m // 2
        vals[tuple(idx)] = 0.0
    return CoefficientTable(dims=q, m=m, values=vals)


def band_multiplier(table: CoefficientTable, nplan: NufftPlan) -> np.ndarray:
    """Compact real band multiplier H_k = Re(c_k) / prod_a psi_hat(k_a/n)^2.

    Shape m^(q-1) x (m/2): all m frequencies (FFT order) on the leading axes,
    k = 0..m/2-1 on the last (the half spectrum of the real transforms; the
    zeroed k = -m/2 plane makes H even, so the other half is implied).
    The (-1)^k signs of the two deconvolutions cancel (nufft.py:149-157).
    """
    q, m = table.dims, table.m
    d2 = nplan.band_deconvolution_squared()
    H = table.values.real.copy()
    for a in range(q):
        shape = [1] * q
        shape[a] = m
        H = H * d2.reshape(shape)
    return np.ascontiguousarray(H[..., : m // 2])


# ---------------------------------------------------------------------------
# device operator


#: operators (device workspace: R x the grids, spectra and band buffers) kept per plan
OPERATOR_CACHE_LIMIT = 8


def _stream_key() -> int:
    """The current CUDA stream: an operator owns mutable workspace (grids, spectra), so
    products issued on different streams get different operators (ak_op: one per stream)."""
    return _torch().cuda.current_stream().cuda_stream


def _cached_operator(cache: dict, key, make):
    """Most-recently-used cache of a plan's operators, at most OPERATOR_CACHE_LIMIT
    (each holds R x ~2 grids of device memory; evicted ones are destroyed)."""
    op = cache.pop(key, None)
    if op is None:
        op = make()
        keys = [k for k in cache if isinstance(k, tuple) and k and k[0] == "op"]
        while len(keys) >= OPERATOR_CACHE_LIMIT:
            del cache[keys.pop(0)]
    cache[key] = op
    return op


class _Operator:
    """ak_op + its coefficient sets: C sets x P windows of (H, scale)."""

    def __init__(self, gs: DeviceGeometry, gi: DeviceGeometry, m: int, R: int,
                 H_host: list, scales: list, per_rhs: bool = False):
        torch = _torch()
        lib = _native.lib()
        self._lib = lib
        P = gs.n_windows
        C = len(H_host)
        self.R, self.C, self.P, self.m = R, C, P, m
        self.per_rhs = per_rhs
        if per_rhs and (C != 1 or len(H_host[0]) != R * P):
            raise ValueError("per-RHS multipliers need one set of R*P tables")
        self.gs, self.gi = gs, gi  # keep geometries alive
        uniq = {}
        self._H = []
        ptrs = []
        for c in range(C):
            for w in range(len(H_host[c])):
                arr = H_host[c][w]
                key = id(arr)
                if key not in uniq:
                    uniq[key] = torch.as_tensor(arr.ravel(), dtype=torch.float64, device="cuda")
                    self._H.append(uniq[key])
                ptrs.append(uniq[key].data_ptr())
        self.hptr = torch.as_tensor(np.asarray(ptrs, dtype=np.int64), device="cuda")
        self.scale = torch.as_tensor(np.asarray(scales, dtype=np.float64).reshape(C * P), device="cuda")
        self._handle = ctypes.c_void_p()
        rc = lib.ak_op_create(gs.handle, gi.handle, m, R, C, _stream_ptr(torch), ctypes.byref(self._handle))
        _native.check(rc, "ak_op_create")

    def apply(self, V, outs: list, sum_windows: list, accumulate: bool = False, flags: int = 0,
              rhs_minor: bool = False) -> None:
        """One product: spread V, transform, interpolate into outs (ak_op_apply).

        RHS-major (default): V (R, N), summed outs (R, N), per-window outs (P, R, N).
        rhs_minor: V (N, R), summed outs (N, R), per-window outs (P, N, R) -- a
        point's R values share a cache line (AK_APPLY_RHS_MINOR)."""
        torch = _torch()
        C = self.C
        optrs = (ctypes.c_void_p * C)(*[o.data_ptr() for o in outs])
        sw = (ctypes.c_int32 * C)(*[1 if s else 0 for s in sum_windows])
        ldo = int(outs[0].shape[-1])
        f = flags | (_native.AK_APPLY_ACCUMULATE if accumulate else 0)
        if self.per_rhs:
            f |= _native.AK_APPLY_H_PER_RHS
        if rhs_minor:
            f |= _native.AK_APPLY_RHS_MINOR
        vptr = V.data_ptr() if V is not None else 0
        ldv = int(V.shape[-1]) if V is not None else (self.R if rhs_minor else self.gs.n_points)
        rc = self._lib.ak_op_apply(self._handle, vptr, ldv, self.hptr.data_ptr(), self.scale.data_ptr(), optrs, ldo,
                                   sw, f, _stream_ptr(torch))
        _native.check(rc, "ak_op_apply")

    def set_rhs_multipliers(self, ptrs) -> None:
        """Replace the per-RHS multiplier table (int64 device tensor of R * P device
        pointers, RHS-major) -- e.g. to re-point a batched operator at a subset of
        cells.  The pointed-to tables must outlive the products that use them."""
        if not self.per_rhs or ptrs.numel() != self.R * self.P:
            raise ValueError("need R * P multiplier pointers of a per-RHS operator")
        self.hptr = ptrs.contiguous()

    def spread_only(self, V) -> None:
        """Zero the op's grids and spread V into them (first half of a point-sharded product)."""
        torch = _torch()
        rc = self._lib.ak_op_apply(self._handle, V.data_ptr(), int(V.shape[-1]), 0, 0, None, 0, None,
                                   _native.AK_APPLY_SPREAD_ONLY, _stream_ptr(torch))
        _native.check(rc, "ak_op_apply(spread only)")

    def spectrum_only(self, V) -> None:
        """Spread V, forward FFT, pack the band spectra into the op's band buffer."""
        torch = _torch()
        rc = self._lib.ak_op_apply(self._handle, V.data_ptr(), int(V.shape[-1]), 0, 0, None, 0, None,
                                   _native.AK_APPLY_SPECTRUM_ONLY, _stream_ptr(torch))
        _native.check(rc, "ak_op_apply(spectrum only)")

    def band(self):
        """The op's compact band spectra (float64 view of complex values): all-reduce buffer."""
        return self._view(self._lib.ak_op_band, "ak_op_band")

    def grids(self):
        """The op's spread grids as a torch CUDA tensor view (all-reduce buffer)."""
        return self._view(self._lib.ak_op_grids, "ak_op_grids")

    def _view(self, fn, what):
        torch = _torch()
        ptr = ctypes.c_void_p()
        count = ctypes.c_int64()
        _native.check(fn(self._handle, ctypes.byref(ptr), ctypes.byref(count)), what)

        class _View:
            __cuda_array_interface__ = {"shape": (int(count.value),), "typestr": "<f8",
                                        "data": (int(ptr.value or 0), False), "version": 3, "strides": None}

        return torch.as_tensor(_View(), device="cuda")

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None and h.value:
            try:
                self._lib.ak_op_destroy(h)
            except Exception:  # pragma: no cover
                pass
            self._handle = None


def _rows_on_device(v, n: int, what: str):
    """(R, n) float64 CUDA tensor from a numpy vector/matrix or a CUDA tensor."""
    torch = _torch()
    if isinstance(v, torch.Tensor):
        t = v.to(device="cuda", dtype=torch.float64)
        on_device = v.is_cuda
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(v, dtype=np.float64)))
        if t.ndim >= 1 and t.shape[-1] == n:
            # page-locked caller buffer (e.g. torch.empty(..., pin_memory=True).numpy()):
            # one stream-ordered DMA, no host sync (the caller's result read syncs later);
            # pageable: one driver-staged copy (measured: 0.46 ms for 8 MB vs 1.2 ms
            # pin-then-copy)
            t = t.to("cuda", non_blocking=t.is_pinned())
        on_device = False
    single = t.ndim == 1
    if t.ndim == 1:
        t = t.reshape(1, -1)
    if t.ndim != 2 or t.shape[1] != n:
        raise ValueError(what)
    return t.contiguous(), single, on_device


def _rhs_minor(Vd):
    """(R, N) device RHS -> (N, R) contiguous (RHS-minor: the layout the kernels gather in
    full sectors).  A caller's tensor that already is the transpose of an (N, R) array is
    used as is."""
    if Vd.stride() == (1, Vd.shape[0]):
        return Vd.t()
    return Vd.t().contiguous()


def _to_caller(t, single: bool, on_device: bool):
    """Device result -> caller: CUDA tensor as is, or a fresh numpy array.

    Host results land in a page-locked buffer from torch's caching host
    allocator (one DMA, no pageable staging copy); the returned array owns it.
    """
    if single:
        t = t[0]
    if on_device:
        return t
    torch = _torch()
    t = t.contiguous()   # RHS-minor results: transposed on the device, then one DMA
    host = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    host.copy_(t, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return host.numpy()


# ---------------------------------------------------------------------------
# plans


@dataclass(frozen=True)
class FastsumPlan:
    """Tables and bin-sorted device geometry bound to one training set
    (fastsum.py:79-102).  ``geometries`` is one DeviceGeometry for all windows."""

    spec: KernelSpec
    window_set: WindowSet
    m: int
    data: Dataset
    nufft_plans: dict = field(repr=False)     # q -> NufftPlan
    tables: dict = field(repr=False)          # q -> CoefficientTable (spec.family)
    geometries: DeviceGeometry = field(repr=False)
    _cache: dict = field(default_factory=dict, repr=False, compare=False)

    @property
    def n_rows(self) -> int:
        return self.data.n_rows

    def table_for(self, window) -> CoefficientTable:
        return self.tables[len(window)]

    def plan_for(self, window) -> NufftPlan:
        return self.nufft_plans[len(window)]

    def eta(self) -> float:
        return self.spec.ell * math.pi * self.m / math.sqrt(2.0)

    # -- coefficient sets -------------------------------------------------
    def _family_set(self, family: str):
        """(per-window H list, per-window scale list) of one kernel family."""
        key = ("set", family)
        hit = self._cache.get(key)
        if hit is None:
            spec = KernelSpec(family, self.spec.ell, self.spec.sigma_f)
            per_q = {}
            for q, nplan in self.nufft_plans.items():
                table = self.tables[q] if family == self.spec.family else kernel_coefficients(
                    family, self.spec.ell, q, self.m)
                per_q[q] = band_multiplier(table, nplan)
            Hs = [per_q[len(w)] for w in self.window_set]
            scales = [spec.operator_scale()] * len(self.window_set)
            hit = (Hs, scales)
            self._cache[key] = hit
        return hit

    def _operator(self, families: tuple, R: int, interp_geom: DeviceGeometry | None = None) -> _Operator:
        gi = interp_geom if interp_geom is not None else self.geometries

        def make():
            sets = [self._family_set(f) for f in families]
            return _Operator(self.geometries, gi, self.m, R, [s[0] for s in sets], [s[1] for s in sets])

        if gi is self.geometries:
            return _cached_operator(self._cache, ("op", families, R, id(gi), _stream_key()), make)
        # cross products (evaluation geometry): keep only the most recent one -- an operator
        # pins its evaluation geometry (weights + workspace), so caching every geometry a
        # caller ever passed would hold their device memory for the plan's lifetime
        key = ("xop", families, R, id(gi), _stream_key())
        op = self._cache.get(key)
        if op is None:
            for k in [k for k in self._cache if isinstance(k, tuple) and k and k[0] == "xop"]:
                del self._cache[k]
            op = make()
            self._cache[key] = op
        return op


def _check_prescaled(data: Dataset, window_set: WindowSet) -> None:
    if data.scaling_state != PRESCALED:
        raise InvalidScalingError("fast summation requires prescaled data")
    if data.d_max is None or max(window_set.lengths) > data.d_max:
        raise InvalidScalingError("data prescaled with a smaller d_max than the longest window")
    if window_set.max_feature() > data.n_features:
        raise ValueError("window refers to a feature beyond the data")


def _eta_warning(ell: float, m: int) -> None:
    eta = ell * math.pi * m / math.sqrt(2.0)
    if eta < 1.0:
        warnings.warn(f"eta = ell*pi*m/sqrt(2) = {eta:.3g} < 1: Fourier approximation "
                      "may be arbitrarily inaccurate for this length-scale", AccuracyWarning, stacklevel=3)


def build_plan(spec: KernelSpec, window_set: WindowSet, preset, data: Dataset, cutoff: int = 6,
               oversampling: float = 2.0, window: str = "kaiser_bessel", features_device=None,
               row_masks=None, tuning=None) -> FastsumPlan:
    """Coefficient tables (host, tiny) + bin-sorted device geometry (fastsum.py:105-133).

    ``features_device`` optionally passes ``data.features`` already resident
    on the GPU (a torch CUDA tensor) to skip the upload.  ``row_masks``
    (windows x rows, bool; extension) restricts each window to a row subset:
    the product is then sum_w K_w restricted to window w's rows (the cell-slab
    multi-GPU layout, distributed.CellShardedPlan).  ``tuning`` (extension) pins
    kernel choices by ak_tuning field name (tests; nufft.DeviceGeometry).
    """
    _check_prescaled(data, window_set)
    m = resolve_m(preset)
    _eta_warning(spec.ell, m)
    lengths = sorted(set(window_set.lengths))
    nufft_plans = {q: NufftPlan(dims=q, m=m, oversampling=oversampling, cutoff=cutoff, window=window)
                   for q in lengths}
    tables = {q: kernel_coefficients(spec.family, spec.ell, q, m) for q in lengths}
    any_plan = nufft_plans[lengths[0]]
    geom = DeviceGeometry(any_plan.n, window_set.lengths, [window_set.columns(w) for w in window_set],
                          data.features if features_device is None else features_device, any_plan.window_fn(),
                          row_masks=row_masks, tuning=tuning)
    return FastsumPlan(spec=spec, window_set=window_set, m=m, data=data, nufft_plans=nufft_plans,
                       tables=tables, geometries=geom)


def fast_matvec(plan: FastsumPlan, v):
    """K v (or the der-family product of a der_* plan), fastsum.py:150-160."""
    V, single, on_dev = _rows_on_device(v, plan.n_rows, "vector length must equal the number of rows")
    if not single:
        raise ValueError("vector length must equal the number of rows")
    torch = _torch()
    out = torch.empty((1, plan.n_rows), dtype=torch.float64, device="cuda")
    plan._operator((plan.spec.family,), 1).apply(V, [out], [True])
    return _to_caller(out, True, on_dev)


def fast_dsigma_matvec(plan: FastsumPlan, v):
    """(dK/d sigma_f) v = (2/sigma_f) K v; a rescale (fastsum.py:163-167)."""
    if DERIVATIVE_PREFACTOR[plan.spec.family] is not None:
        raise ValueError("sigma_f derivative applies to the base kernel plan")
    return (2.0 / plan.spec.sigma_f) * fast_matvec(plan, v)


def fast_matvecs(plan: FastsumPlan, V, dell: bool = False, dsigma: bool = False) -> dict:
    """Batched products for R right-hand sides sharing one spread per window.

    Returns {"K": K V, "dK_dell": dK/d ell V, "dK_dsigma": dK/d sigma_f V}
    (the last two only when asked), each shaped like V.  ``dell`` needs a
    base-family plan; it equals fast_matvec on the reference's der_* plan.
    """
    if dell and DERIVATIVE_PREFACTOR[plan.spec.family] is not None:
        raise ValueError("derivative sets need a base-family plan")
    Vd, single, on_dev = _rows_on_device(V, plan.n_rows, "V must be (N,) or (R, N)")
    torch = _torch()
    R = Vd.shape[0]
    fams = (plan.spec.family,) + ((DERIVATIVE_FAMILY[plan.spec.family],) if dell else ())
    if R > 1:
        # RHS-minor products; device results are (R, N) views of the (N, R) outputs
        outs = [torch.empty((plan.n_rows, R), dtype=torch.float64, device="cuda") for _ in fams]
        plan._operator(fams, R).apply(_rhs_minor(Vd), outs, [True] * len(fams), rhs_minor=True)
        outs = [o.t() for o in outs]
    else:
        outs = [torch.empty((R, plan.n_rows), dtype=torch.float64, device="cuda") for _ in fams]
        plan._operator(fams, R).apply(Vd, outs, [True] * len(fams))
    res = {"K": _to_caller(outs[0], single, on_dev)}
    if dell:
        res["dK_dell"] = _to_caller(outs[1], single, on_dev)
    if dsigma:
        if DERIVATIVE_PREFACTOR[plan.spec.family] is not None:
            raise ValueError("sigma_f derivative applies to the base kernel plan")
        res["dK_dsigma"] = _to_caller(outs[0] * (2.0 / plan.spec.sigma_f), single, on_dev)
    return res


def prepare_eval_points(plan: FastsumPlan, data: Dataset) -> DeviceGeometry:
    """Device geometry of out-of-sample nodes, same windows (fastsum.py:170-177)."""
    if data.scaling_state != PRESCALED or not same_scaling(plan.data, data):
        raise ScalingMismatchError("evaluation data must be prescaled with the training maps")
    ws = plan.window_set
    any_plan = next(iter(plan.nufft_plans.values()))
    return DeviceGeometry(any_plan.n, ws.lengths, [ws.columns(w) for w in ws], data.features,
                          any_plan.window_fn(), tuning=plan.geometries.tuning)


def fast_cross_matvec(plan: FastsumPlan, eval_geoms: DeviceGeometry, v, n_eval: int):
    """K(eval, train) v: spread at the training nodes, interp at the eval nodes
    (fastsum.py:180-191)."""
    V, single, on_dev = _rows_on_device(v, plan.n_rows, "vector length must equal the number of training rows")
    if eval_geoms.n_points != n_eval:
        raise ValueError("n_eval does not match the evaluation geometry")
    torch = _torch()
    out = torch.empty((1, n_eval), dtype=torch.float64, device="cuda")
    plan._operator((plan.spec.family,), 1, eval_geoms).apply(V, [out], [True])
    return _to_caller(out, True, on_dev)


# ---------------------------------------------------------------------------
# mixed-kernel plans (per-window family and length-scale)


@dataclass(frozen=True)
class MixedKernelPlan:
    """Additive kernel with a per-window family and length-scale.

    One reference plan cannot express this; its oracle is the
    sum of single-window reference plans.  All windows share sigma_f.
    """

    specs: tuple
    window_set: WindowSet
    m: int
    data: Dataset
    nufft_plans: dict = field(repr=False)
    geometries: DeviceGeometry = field(repr=False)
    _cache: dict = field(default_factory=dict, repr=False, compare=False)

    @property
    def n_rows(self) -> int:
        return self.data.n_rows

    @property
    def sigma_f(self) -> float:
        return self.specs[0].sigma_f

    def _sets(self):
        hit = self._cache.get("sets")
        if hit is None:
            Hk, Hd, sk, sd = [], [], [], []
            for spec, w in zip(self.specs, self.window_set):
                q = len(w)
                nplan = self.nufft_plans[q]
                Hk.append(band_multiplier(kernel_coefficients(spec.family, spec.ell, q, self.m), nplan))
                der = spec.derivative()
                Hd.append(band_multiplier(kernel_coefficients(der.family, der.ell, q, self.m), nplan))
                sk.append(spec.operator_scale())
                sd.append(der.operator_scale())
            hit = ((Hk, sk), (Hd, sd))
            self._cache["sets"] = hit
        return hit

    def _operator(self, R: int, dell: bool) -> _Operator:
        def make():
            (Hk, sk), (Hd, sd) = self._sets()
            H = [Hk, Hd] if dell else [Hk]
            S = [sk, sd] if dell else [sk]
            return _Operator(self.geometries, self.geometries, self.m, R, H, S)

        return _cached_operator(self._cache, ("op", R, dell, _stream_key()), make)


def build_mixed_plan(specs, window_set: WindowSet, preset, data: Dataset, cutoff: int = 6,
                     oversampling: float = 2.0, window: str = "kaiser_bessel",
                     features_device=None, row_masks=None, tuning=None) -> MixedKernelPlan:
    specs = tuple(specs)
    if len(specs) != len(window_set):
        raise ValueError("need one KernelSpec per window")
    for s in specs:
        if DERIVATIVE_PREFACTOR[s.family] is not None:
            raise ValueError("mixed plans take base families; derivatives are computed alongside")
    if len({s.sigma_f for s in specs}) != 1:
        raise ValueError("all windows must share sigma_f")
    _check_prescaled(data, window_set)
    m = resolve_m(preset)
    for s in specs:
        _eta_warning(s.ell, m)
    lengths = sorted(set(window_set.lengths))
    nufft_plans = {q: NufftPlan(dims=q, m=m, oversampling=oversampling, cutoff=cutoff, window=window)
                   for q in lengths}
    any_plan = nufft_plans[lengths[0]]
    geom = DeviceGeometry(any_plan.n, window_set.lengths, [window_set.columns(w) for w in window_set],
                          data.features if features_device is None else features_device, any_plan.window_fn(),
                          row_masks=row_masks, tuning=tuning)
    return MixedKernelPlan(specs=specs, window_set=window_set, m=m, data=data, nufft_plans=nufft_plans,
                           geometries=geom)


def mixed_matvecs(plan: MixedKernelPlan, V, dell: bool = True, dsigma: bool = True) -> dict:
    """K V, the per-window dK/d ell_w V (shape (P, R, N)) and dK/d sigma_f V."""
    Vd, single, on_dev = _rows_on_device(V, plan.n_rows, "V must be (N,) or (R, N)")
    torch = _torch()
    R, N, P = Vd.shape[0], plan.n_rows, len(plan.window_set)
    minor = R > 1
    if minor:
        # RHS-minor products: K (N, R), per-window dK/dl_w (P, N, R); returned as
        # (R, N) / (P, R, N) views on the device
        outs = [torch.empty((N, R), dtype=torch.float64, device="cuda")]
        if dell:
            outs.append(torch.empty((P, N, R), dtype=torch.float64, device="cuda"))
        plan._operator(R, dell).apply(_rhs_minor(Vd), outs, [True, False][: len(outs)], rhs_minor=True)
        outs = [outs[0].t()] + ([outs[1].permute(0, 2, 1)] if dell else [])
    else:
        outs = [torch.empty((R, N), dtype=torch.float64, device="cuda")]
        if dell:
            outs.append(torch.empty((P, R, N), dtype=torch.float64, device="cuda"))
        plan._operator(R, dell).apply(Vd, outs, [True, False][: len(outs)])
    res = {"K": _to_caller(outs[0], single, on_dev)}
    if dell:
        d = outs[1][:, 0] if single else outs[1]
        res["dK_dell"] = d if on_dev else d.contiguous().cpu().numpy()
    if dsigma:
        res["dK_dsigma"] = _to_caller(outs[0] * (2.0 / plan.sigma_f), single, on_dev)
    return res
