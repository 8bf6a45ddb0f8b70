"""ORACLE -- TEST INFRASTRUCTURE ONLY.

Full-size oracle products for the BASELINE configurations (C3, C4, C5 at
their real N), used by tests/test_gpu_fullsize.py and by bench.py's
post-timing ``rel_err_vs_oracle`` extras.  The product package never imports
this module.

The arithmetic is restate.py's (the reference's own path:
/root/reference/pkg/src/addkern/fastsum.py:150-160 per window,
nufft.py:169-394 underneath); this module only organises it so full-size
checks finish in tens of seconds on the host's threads and bounded RAM:

* windows are processed ONE AT A TIME (a 3-D window's geometry at N = 4M is
  1.25 GB of tap weights; config 5 has ten windows);
* each window's rows are split into row chunks, one Geometry per chunk,
  gridded by a thread pool (ctypes releases the GIL in the C loops); the
  chunks' grids are summed before the transform (the gridding is linear);
* one spread + forward transform per (window, RHS) serves every coefficient
  set of that window (K and dK/d ell), as in the reference each set is
  c_hat * type1(v) -> type2 (fastsum.py:157-159) with its own scale
  (fastsum.py:136-138).

The window sum, scale and real part follow fastsum.py:150-160 (scale applied
after the window sum is equal up to rounding to the per-window scale used
here: all windows of a set share it, except config 5 whose reference is a
sum of single-window plans anyway).
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import restate as R


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def window_products(X, cols, sets, V, pool, chunks, m=32, cutoff=6, oversampling=2.0):
    """Products of ONE window for every coefficient set and RHS.

    X     (N, d) prescaled features; cols: 0-based feature columns of the window
    sets  list of (family, ell, sigma_f): one reference single-window plan each
          (KernelSpec(family, ell, sigma_f), WindowSet((w,)), fastsum.py:105-133)
    V     (R, N) real right-hand sides
    Returns a list over sets of (R, N) float64 arrays: scale * Re type2(c_hat * type1(v)).
    """
    cols = list(cols)
    q = len(cols)
    plan = R.Nufft(q, m, oversampling, cutoff)
    N = X.shape[0]
    b = np.linspace(0, N, chunks + 1).astype(np.int64)
    rng = range(chunks)
    sub = list(pool.map(lambda c: R.Geometry(plan, np.ascontiguousarray(X[b[c]:b[c + 1]][:, cols])), rng))
    tables = [R.kernel_coefficients(fam, ell, q, m) for fam, ell, _ in sets]
    scales = [R.operator_scale(fam, ell, sf) for fam, ell, sf in sets]
    V = np.atleast_2d(np.asarray(V, dtype=np.float64))
    outs = [np.empty((V.shape[0], N)) for _ in sets]
    for r in range(V.shape[0]):
        v = V[r].astype(np.complex128)
        grids = list(pool.map(lambda c: R.spread_grid(plan, sub[c], v[b[c]:b[c + 1]]), rng))
        grid = grids[0]
        for g in grids[1:]:
            grid = grid + g
        S = R.band_spectrum(plan, grid)
        for s, (tab, sc) in enumerate(zip(tables, scales)):
            g = R.type2_grid(plan, tab * S)
            parts = list(pool.map(lambda c: R.interp_grid(plan, sub[c], g), rng))
            outs[s][r] = sc * np.concatenate(parts).real
    return outs


def products(X, windows, specs, V, dell=False, per_window_dell=False, threads=None, chunks=None):
    """Additive products over windows, each window its own reference plan.

    windows  0-based column tuples; specs: (family, ell, sigma_f) per window (base families)
    V        (R, N) right-hand sides
    dell     also dK/d ell (each window's derivative family, same ell)
    per_window_dell  keep dK/d ell_w per window (config 5: shape (P, R, N))
    Returns {"K": (R, N), "dK_dell": (R, N) or (P, R, N)}; dK/d sigma_f is
    (2/sigma_f) K (fastsum.py:163-167) and is derived by the caller.
    """
    threads = threads or host_threads()
    chunks = chunks or threads
    X = np.asarray(X, dtype=np.float64)
    V = np.atleast_2d(np.asarray(V, dtype=np.float64))
    N = X.shape[0]
    K = np.zeros((V.shape[0], N))
    dK = None
    if dell:
        dK = np.zeros((len(windows), V.shape[0], N)) if per_window_dell else np.zeros((V.shape[0], N))
    with ThreadPoolExecutor(max_workers=threads) as pool:
        for k, (cols, (fam, ell, sf)) in enumerate(zip(windows, specs)):
            sets = [(fam, ell, sf)]
            if dell:
                sets.append((R.DERIVATIVE_FAMILY[fam], ell, sf))
            outs = window_products(X, cols, sets, V, pool, chunks)
            K += outs[0]
            if dell:
                if per_window_dell:
                    dK[k] = outs[1]
                else:
                    dK += outs[1]
            del outs
    res = {"K": K}
    if dell:
        res["dK_dell"] = dK
    return res


def config_products(wl, rhs=None, dell=False, per_window_dell=False, threads=None, chunks=None):
    """products() of a configs.Workload at its full size (rhs: indices of wl.V, default all)."""
    V = wl.V if rhs is None else wl.V[list(rhs)]
    windows = [wl.window_set.columns(w) for w in wl.window_set]
    specs = [(s.family, s.ell, s.sigma_f) for s in wl.specs]
    return products(wl.data.features, windows, specs, V, dell=dell, per_window_dell=per_window_dell,
                    threads=threads, chunks=chunks)


def rel_err(a, b) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))


def max_rel_rows(a, b) -> float:
    """Max over the leading index of the per-vector relative l2 error."""
    a = np.asarray(a).reshape(-1, np.asarray(a).shape[-1])
    b = np.asarray(b).reshape(-1, np.asarray(b).shape[-1])
    return max(rel_err(x, y) for x, y in zip(a, b))
