"""Seeded synthetic workloads for the five BASELINE.json configurations.

The UCI datasets behind the paper's experiments are not available; these
generators reproduce the shapes and distributions BASELINE.json names
(SURVEY.md §8d).  Seeds: features default_rng(1000+c), right-hand sides
default_rng(2000+c), per-window length-scales default_rng(3000+c).  Raw
features go through zscore -> quarter box -> prescale(d_max) exactly like the
reference pipeline, and quarter-box length-scales become ell / sqrt(d_max).
``n`` overrides the row count (small parity cases with the same distribution).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .dataset import from_arrays, minmax_to_quarter_box, prescale, zscore_normalize
from .kernels import KernelSpec
from .windows import WindowSet, consec_windows


@dataclass
class Workload:
    name: str
    data: object                # prescaled Dataset
    window_set: WindowSet
    specs: tuple                # one base-family KernelSpec per window (prescaled ell)
    V: np.ndarray               # (R, N) right-hand sides
    dell: bool                  # the config asks for dK/d ell products
    dsigma: bool                # ... and dK/d sigma_f
    mixed: bool                 # per-window family / ell (needs a MixedKernelPlan)

    @property
    def spec(self) -> KernelSpec:
        return self.specs[0]


def _prescaled(X: np.ndarray, d_max: int):
    ds = from_arrays(X, np.zeros(X.shape[0]))
    ds = minmax_to_quarter_box(zscore_normalize(ds))
    out, _ = prescale(ds, d_max, 1.0)
    return out


def config1(n: int = 2000) -> Workload:
    """Gaussian, N=2k, d=9 iid U[-1,1], 3 windows of 3, ell=1, sigma_f=1, 1 RHS."""
    X = np.random.default_rng(1001).uniform(-1.0, 1.0, size=(n, 9))
    ds = _prescaled(X, 3)
    ws = consec_windows(9, 3)
    spec = KernelSpec("gauss", 1.0 / math.sqrt(3.0), 1.0)
    V = np.random.default_rng(2001).normal(size=(1, n))
    return Workload("C1", ds, ws, (spec,) * len(ws), V, False, False, False)


def config2(n: int = 20000) -> Workload:
    """Matern(1/2), N=20k, d=8 iid N(0,1), 4 windows of 2, ell=0.5; K, dK/dl, dK/ds."""
    X = np.random.default_rng(1002).normal(size=(n, 8))
    ds = _prescaled(X, 2)
    ws = consec_windows(8, 2)
    spec = KernelSpec("matern12", 0.5 / math.sqrt(2.0), 1.0)
    V = np.random.default_rng(2002).normal(size=(1, n))
    return Workload("C2", ds, ws, (spec,) * len(ws), V, True, True, False)


def config3(n: int = 100000) -> Workload:
    """Gaussian, N=100k, d=12 iid U[-1,1], 4 windows of 3, ell=2, 8 RHS, + dK/dl."""
    X = np.random.default_rng(1003).uniform(-1.0, 1.0, size=(n, 12))
    ds = _prescaled(X, 3)
    ws = consec_windows(12, 3)
    spec = KernelSpec("gauss", 2.0 / math.sqrt(3.0), 1.0)
    V = np.random.default_rng(2003).normal(size=(8, n))
    return Workload("C3", ds, ws, (spec,) * len(ws), V, True, False, False)


def config4(n: int = 1_000_000) -> Workload:
    """Gaussian, N=1M, d=30 5-component mixture (means U[-1,1], std 0.3), 10 windows of 3."""
    rng = np.random.default_rng(1004)
    means = rng.uniform(-1.0, 1.0, size=(5, 30))
    comp = rng.integers(0, 5, size=n)
    X = means[comp] + 0.3 * rng.normal(size=(n, 30))
    ds = _prescaled(X, 3)
    ws = consec_windows(30, 3)
    spec = KernelSpec("gauss", 1.0 / math.sqrt(3.0), 1.0)
    V = np.random.default_rng(2004).normal(size=(1, n))
    return Workload("C4", ds, ws, (spec,) * len(ws), V, False, False, False)


C5_LENGTHS = (3, 3, 3, 3, 3, 3, 2, 2, 1, 1)


def config5(n: int = 4_000_000, rhs: int = 16) -> Workload:
    """Mixed kernels, N=4M, d=24 MVN (pairwise corr 0.5), windows [3x6, 2x2, 1x2],
    Gaussian on 3-D windows and Matern(1/2) elsewhere, ell_w ~ U[0.5, 3], 16 RHS,
    K V + all dK/d ell_w V + dK/d sigma_f V."""
    rng = np.random.default_rng(1005)
    # Sigma = 0.5 I + 0.5 11^T  <=>  x = sqrt(.5) z + sqrt(.5) s 1 with one shared factor s
    common = rng.normal(size=(n, 1))
    X = math.sqrt(0.5) * rng.normal(size=(n, 24)) + math.sqrt(0.5) * common
    ds = _prescaled(X, 3)
    wins, start = [], 1
    for q in C5_LENGTHS:
        wins.append(tuple(range(start, start + q)))
        start += q
    ws = WindowSet(tuple(wins), d_max=3)
    ells = np.random.default_rng(3005).uniform(0.5, 3.0, size=len(wins))
    specs = tuple(KernelSpec("gauss" if len(w) == 3 else "matern12", float(l) / math.sqrt(3.0), 1.0)
                  for w, l in zip(wins, ells))
    V = np.random.default_rng(2005).normal(size=(rhs, n))
    return Workload("C5", ds, ws, specs, V, True, True, True)


CONFIGS = {"C1": config1, "C2": config2, "C3": config3, "C4": config4, "C5": config5}
