"""ORACLE -- TEST INFRASTRUCTURE ONLY.

The paper's analytic Fourier-error bounds (arXiv 2404.17344, Theorems 3.2 /
3.3), restated from the reference's
/root/reference/pkg/src/addkern/bounds.py:56-130 for the acceptance checks
the north_star asks for ("within the paper's error bound of the exact dense
additive-kernel matvec at N <= 20k").  Pinned against values the unmodified
reference produced (tests/golden/bounds.npz, tests/golden/make_golden.py).

With eta = ell * pi * m / sqrt(2) (ell in prescaled units, m modes per axis),
valid for eta >= 1, the worst-case error of the (truncated, FFT-sampled)
Fourier approximation of one window kernel kappa_s is at most
analytic_bound(family, q, ell, m); the per-entry matvec error is then
(Hoelder)

    |(K v)_i - (K~ v)_i| <= sigma_f^2 * pre * sum_s ||v||_1 * bound_s ,

pre = 1 (gauss) or 2/ell (der_gauss, the derivative family's unit-scale
operator factor, fastsum.py:136-138).  Bounds exist for gauss / der_gauss at
q in {1, 3} only.
"""

from __future__ import annotations

import math

ELL_STAR = 0.5 * math.sqrt(2.0 / (5.0 + math.sqrt(17.0)))   # bounds.py:31: branch point of the der terms
_S2PI = math.sqrt(2.0 * math.pi)
_SPI = math.sqrt(math.pi)


class EtaTooSmall(ValueError):
    """eta < 1: the theorems do not apply (reference EtaTooSmallError, bounds.py:53-56)."""


def eta(ell: float, m: int) -> float:
    """bounds.py:49-51."""
    return ell * math.pi * m / math.sqrt(2.0)


def _checked(ell: float, m: int) -> float:
    if ell <= 0:
        raise ValueError("ell must be positive")                     # bounds.py:42-44
    if m < 2 or m % 2:
        raise ValueError("m must be even and >= 2")                   # bounds.py:45-46
    e = eta(ell, m)
    if e < 1.0:
        raise EtaTooSmall(f"eta = {e:.4g} < 1")
    return e


def gamma_term(ell, m):
    """|c_{m/2}| bound of the Gaussian (bounds.py:59-66)."""
    e = _checked(ell, m)
    head = ell * _S2PI * math.exp(-e * e)
    tail = math.exp(-1.0 / (8.0 * ell * ell)) if ell < 0.5 else 2.0 * ell * math.exp(-0.5)
    return head + tail / (e * e)


def a_term(ell, m):
    """Tail sum bound of the Gaussian's coefficients beyond m/2 (bounds.py:69-76)."""
    e = _checked(ell, m)
    head = math.exp(-e * e) / (2.0 * e * _SPI)
    if ell < 0.5:
        return head + math.exp(-1.0 / (8.0 * ell * ell)) / (math.sqrt(2.0) * ell * math.pi * e)
    return head + math.sqrt(2.0) * math.exp(-0.5) / (math.pi * e)


def xi_term(ell, m):
    """|c_{m/2}| bound of the derivative Gaussian (bounds.py:79-86)."""
    e = _checked(ell, m)
    head = (e * e + 0.5) * ell * _S2PI * math.exp(-e * e)
    if ell <= ELL_STAR:
        return head + math.exp(-1.0 / (8.0 * ell * ell)) / (8.0 * e * e * ell * ell)
    return head + 1.0 / (e * e) + 3.0 * ell / (2.0 * e * e)


def s_term(ell, m):
    """Tail sum bound of the derivative Gaussian (bounds.py:89-100)."""
    e = _checked(ell, m)
    x = math.exp(-e * e)
    head = math.erfc(e) / 4.0 + e * x / (2.0 * _SPI) + x / (4.0 * _SPI * e)
    if ell <= ELL_STAR:
        return head + math.exp(-1.0 / (8.0 * ell * ell)) / (8.0 * math.sqrt(2.0) * math.pi * ell ** 3 * e)
    return head + 1.0 / (math.sqrt(2.0) * math.pi * ell * e) + 3.0 / (2.0 * math.sqrt(2.0) * math.pi * e)


def analytic_bound(family: str, q: int, ell: float, m: int) -> float:
    """Theorem 3.2 (gauss) / 3.3 (der_gauss) for q = 3, and the 1-D forms
    (bounds.py:103-130)."""
    if family not in ("gauss", "der_gauss"):
        raise ValueError("bounds exist for the gauss and der_gauss families only")
    if q not in (1, 3):
        raise ValueError("bounds exist for window lengths 1 and 3 only")
    g, a = gamma_term(ell, m), a_term(ell, m)
    if family == "gauss":
        return 2.0 * g + 4.0 * a if q == 1 else 15.0 * g * (g + 2.5) + 102.0 * a
    xi, s = xi_term(ell, m), s_term(ell, m)
    if q == 1:
        return 2.0 * xi + 4.0 * s
    return (2.5 * xi + 15.0 * g) * (15.0 + 12.0 * g) + 75.0 * s + 6.0 * a * (23.2 * s + 87.0)


def per_entry_bound(family: str, windows_q, ell: float, m: int, sigma_f: float, v) -> float:
    """sigma_f^2 * pre * sum_s ||v||_1 * bound_s: the bound on
    max_i |(K v)_i - (K~ v)_i| for the additive kernel over the given windows."""
    import numpy as np

    pre = 1.0 if family == "gauss" else 2.0 / ell
    l1 = float(np.abs(np.asarray(v, dtype=np.float64)).sum())
    return sigma_f ** 2 * pre * l1 * sum(analytic_bound(family, q, ell, m) for q in windows_q)
