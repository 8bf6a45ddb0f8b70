"""Kernel setup: families, hyperparameters and the radial profiles.

Mirrors /root/reference/pkg/src/addkern/kernels.py:28-78:

    gauss         exp(-r^2 / (2 ell^2))
    der_gauss     t exp(-t),  t = r^2 / (2 ell^2)       (operator factor 2/ell)
    matern12      exp(-r / ell)
    der_matern12  t exp(-t),  t = r / ell               (operator factor 1/ell)

so that  dK/d ell = sigma_f^2 * sum_s (pre/ell) K_s^der  (PAPER.md:359-367,
1402-1424), with ell always in the prescaled units of the data.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

GAUSS = "gauss"
DER_GAUSS = "der_gauss"
MATERN12 = "matern12"
DER_MATERN12 = "der_matern12"

FAMILIES = (GAUSS, DER_GAUSS, MATERN12, DER_MATERN12)

#: per-window operator factor on top of sigma_f^2 (None = plain kernel)
DERIVATIVE_PREFACTOR = {GAUSS: None, DER_GAUSS: 2.0, MATERN12: None, DER_MATERN12: 1.0}

#: the plain kernel underlying each family
BASE_FAMILY = {GAUSS: GAUSS, DER_GAUSS: GAUSS, MATERN12: MATERN12, DER_MATERN12: MATERN12}

#: the ell-derivative family of each plain kernel
DERIVATIVE_FAMILY = {GAUSS: DER_GAUSS, MATERN12: DER_MATERN12}

DENSE_ROW_LIMIT = 20_000


@dataclass(frozen=True)
class KernelSpec:
    """Kernel family plus hyperparameters (ell in prescaled units)."""

    family: str
    ell: float
    sigma_f: float = 1.0

    def __post_init__(self):
        if self.family not in FAMILIES:
            raise ValueError(f"unknown kernel family {self.family!r}")
        if not self.ell > 0:
            raise ValueError("ell must be positive")
        if not self.sigma_f > 0:
            raise ValueError("sigma_f must be positive")

    def base(self) -> "KernelSpec":
        return KernelSpec(BASE_FAMILY[self.family], self.ell, self.sigma_f)

    def derivative(self) -> "KernelSpec":
        """The dK/d ell spec of a plain kernel (der_* family, same ell, sigma_f)."""
        base = BASE_FAMILY[self.family]
        return KernelSpec(DERIVATIVE_FAMILY[base], self.ell, self.sigma_f)

    def operator_scale(self) -> float:
        """sigma_f^2 * (1 | pre/ell), applied after the window sum (fastsum.py:136-138)."""
        pre = DERIVATIVE_PREFACTOR[self.family]
        s2 = self.sigma_f * self.sigma_f
        return s2 if pre is None else s2 * (pre / self.ell)


def radial_profile(family: str, ell: float, r2) -> np.ndarray:
    """Unit-scale radial kernel evaluated on squared distances r2."""
    r2 = np.asarray(r2, dtype=np.float64)
    if family == GAUSS:
        return np.exp(-r2 / (2.0 * ell * ell))
    if family == DER_GAUSS:
        u = r2 / (2.0 * ell * ell)
        return u * np.exp(-u)
    if family == MATERN12:
        return np.exp(-np.sqrt(r2) / ell)
    if family == DER_MATERN12:
        u = np.sqrt(r2) / ell
        return u * np.exp(-u)
    raise ValueError(f"unknown kernel family {family!r}")


def eval_kernel(spec: KernelSpec, arg: float) -> float:
    """One kernel value; ``arg`` is r^2 for the gauss families and r for matern."""
    if arg < 0:
        raise ValueError("distance argument must be nonnegative")
    r2 = arg if spec.family in (GAUSS, DER_GAUSS) else arg * arg
    return float(radial_profile(spec.family, spec.ell, r2))


# ---------------------------------------------------------------------------
# exact dense products on the GPU (kernels.py:92-170 of the reference)


def _check_limit(*sizes) -> None:
    from .errors import DenseLimitExceededError

    for n in sizes:
        if n > DENSE_ROW_LIMIT:
            raise DenseLimitExceededError(f"{n} rows exceeds the dense limit of {DENSE_ROW_LIMIT}")


def _dense(spec: KernelSpec, ws, Xa, Xb, v=None, matrix=False):
    import ctypes

    import torch

    from . import _native
    from .nufft import _stream_ptr, _torch

    _torch()
    lib = _native.lib()
    A = torch.as_tensor(np.ascontiguousarray(Xa, dtype=np.float64), device="cuda")
    B = A if Xb is Xa else torch.as_tensor(np.ascontiguousarray(Xb, dtype=np.float64), device="cuda")
    P = len(ws)
    q = (ctypes.c_int32 * P)(*ws.lengths)
    flat = []
    for w in ws:
        c = ws.columns(w)
        flat.extend(c + [0] * (3 - len(c)))
    cols = (ctypes.c_int32 * (3 * P))(*flat)
    fam = _native.FAMILY_CODE[spec.family]
    scale = spec.operator_scale()
    st = _stream_ptr(torch)
    if matrix:
        M = torch.empty((A.shape[0], B.shape[0]), dtype=torch.float64, device="cuda")
        _native.check(lib.ak_dense_apply(fam, spec.ell, scale, P, q, cols, A.data_ptr(), A.shape[0], A.shape[1],
                                         B.data_ptr(), B.shape[0], B.shape[1], 0, 0, M.data_ptr(), st),
                      "ak_dense_apply")
        return M.cpu().numpy()
    vd = torch.as_tensor(np.ascontiguousarray(v, dtype=np.float64), device="cuda")
    out = torch.empty(A.shape[0], dtype=torch.float64, device="cuda")
    _native.check(lib.ak_dense_apply(fam, spec.ell, scale, P, q, cols, A.data_ptr(), A.shape[0], A.shape[1],
                                     B.data_ptr(), B.shape[0], B.shape[1], vd.data_ptr(), out.data_ptr(), 0, st),
                  "ak_dense_apply")
    return out.cpu().numpy()


def dense_matvec(spec: KernelSpec, ws, X, v) -> np.ndarray:
    """Exact sigma_f^2 * pre * sum_s K_s v on the GPU (reference kernels.py:123-137)."""
    v = np.asarray(v, dtype=np.float64)
    if v.shape != (X.n_rows,):
        raise ValueError("vector length must equal the number of rows")
    _check_limit(X.n_rows)
    return _dense(spec, ws, X.features, X.features, v)


def dense_cross_matvec(spec: KernelSpec, ws, X_eval, X_train, v) -> np.ndarray:
    """K(X_eval, X_train) v with dense_matvec's scaling (reference kernels.py:140-151)."""
    v = np.asarray(v, dtype=np.float64)
    if v.shape != (X_train.n_rows,):
        raise ValueError("vector length must equal the number of training rows")
    _check_limit(X_eval.n_rows, X_train.n_rows)
    return _dense(spec, ws, X_eval.features, X_train.features, v)


def dsigma_matvec(spec: KernelSpec, ws, X, v) -> np.ndarray:
    """(dK/d sigma_f) v = (2/sigma_f) K v of the base family (reference kernels.py:154-156)."""
    return (2.0 / spec.sigma_f) * dense_matvec(spec.base(), ws, X, v)


def dense_matrix(spec: KernelSpec, ws, X) -> np.ndarray:
    """The full operator (diagnostics, small N; reference kernels.py:159-170)."""
    _check_limit(X.n_rows)
    return _dense(spec, ws, X.features, X.features, matrix=True)
