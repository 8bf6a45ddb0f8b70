"""GPU parity: the CUDA path (through libaddkern_b200's C ABI) against the
reference's golden vectors and the CPU oracle.

Tolerance (north_star): relative l2 <= 1e-8 in float64 against the
reference's own NFFT matvec on the same inputs.  Expected ~1e-13: both sides
carry the same NUFFT (error ~1e-12 vs the exact trig sum) and differ only by
rounding and the ~1e-14 window polynomial.
"""

import math

import numpy as np
import pytest

from conftest import golden, rel

pytestmark = pytest.mark.gpu

TOL = 1e-8


def _ds(X, d_max):
    from paper_2404_17344_b200.dataset import PRESCALED, Dataset

    return Dataset(X, np.zeros(X.shape[0]), tuple(f"x{i + 1}" for i in range(X.shape[1])),
                   scaling_state=PRESCALED, d_max=int(d_max))


def _ws(g):
    from paper_2404_17344_b200.windows import WindowSet

    return WindowSet(tuple(tuple(int(c) for c in row[:q]) for row, q in zip(g["windows"], g["lengths"])),
                     d_max=int(g["d_max"]))


def _plan(g, family=None, preset="default", **kw):
    from paper_2404_17344_b200.fastsum import build_plan
    from paper_2404_17344_b200.kernels import KernelSpec

    spec = KernelSpec(family or str(g["families"][0]), float(g["ells"][0]), float(g["sigma_f"]))
    return build_plan(spec, _ws(g), preset, _ds(g["X"], g["d_max"]), **kw)


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4"])
def test_configs_match_reference(cuda, name):
    from paper_2404_17344_b200.fastsum import fast_dsigma_matvec, fast_matvec, fast_matvecs

    g = golden(name)
    plan = _plan(g)
    for r, v in enumerate(g["V"]):
        assert rel(fast_matvec(plan, v), g["K_default"][r]) <= TOL
    res = fast_matvecs(plan, g["V"], dell="dK_dell_default" in g, dsigma="dK_dsigma_default" in g)
    assert rel(res["K"], g["K_default"]) <= TOL
    if "dK_dell_default" in g:
        assert rel(res["dK_dell"], g["dK_dell_default"]) <= TOL
        dplan = _plan(g, family="der_" + str(g["families"][0]))
        for r, v in enumerate(g["V"]):
            assert rel(fast_matvec(dplan, v), g["dK_dell_default"][r]) <= TOL
    if "dK_dsigma_default" in g:
        assert rel(res["dK_dsigma"], g["dK_dsigma_default"]) <= TOL
        assert rel(fast_dsigma_matvec(plan, g["V"][0]), g["dK_dsigma_default"][0]) <= TOL
    if "K_dense" in g:
        # both fast paths carry the same Fourier error against the exact dense sum
        ref_err = rel(g["K_default"], g["K_dense"])
        gpu_err = rel(res["K"], g["K_dense"])
        assert abs(gpu_err - ref_err) <= 1e-8


def test_mixed_c5_matches_sum_of_reference_plans(cuda):
    from paper_2404_17344_b200.fastsum import build_mixed_plan, mixed_matvecs
    from paper_2404_17344_b200.kernels import KernelSpec

    g = golden("c5")
    specs = [KernelSpec(str(f), float(l), 1.0) for f, l in zip(g["families"], g["ells"])]
    plan = build_mixed_plan(specs, _ws(g), "default", _ds(g["X"], g["d_max"]))
    res = mixed_matvecs(plan, g["V"])
    assert rel(res["K"], g["K_default"]) <= TOL
    assert rel(res["dK_dsigma"], g["dK_dsigma_default"]) <= TOL
    for w in range(len(specs)):
        assert rel(res["dK_dell"][w], g["dK_dell_default"][w]) <= TOL


def test_presets_match_reference(cuda):
    g = golden("c1_presets")
    from paper_2404_17344_b200.fastsum import fast_matvec

    for preset in ("rough", "fine"):
        assert rel(fast_matvec(_plan(g, preset=preset), g["V"][0]), g[f"K_{preset}"][0]) <= TOL


def test_family_ell_preset_grid(cuda):
    """Reference test_fastsum.py:62-84 grid: 4 families x ell {0.1,1,10} x 3 presets."""
    from paper_2404_17344_b200.fastsum import build_plan, fast_matvec
    from paper_2404_17344_b200.kernels import KernelSpec
    from paper_2404_17344_b200.windows import WindowSet

    g = golden("family_grid")
    ds = _ds(g["X"], 3)
    ws = WindowSet(((1, 2, 3), (4, 5, 6)), d_max=3)
    for fam in ("gauss", "der_gauss", "matern12", "der_matern12"):
        for ell in (0.1, 1.0, 10.0):
            for preset in ("rough", "default", "fine"):
                plan = build_plan(KernelSpec(fam, ell, math.sqrt(0.5)), ws, preset, ds)
                assert rel(fast_matvec(plan, g["v"]), g[f"{fam}_{ell}_{preset}"]) <= TOL, (fam, ell, preset)


@pytest.mark.parametrize("q", [1, 2, 3])
@pytest.mark.parametrize("m", [8, 16])
def test_nufft_type1_type2_match_reference(cuda, q, m):
    from paper_2404_17344_b200.nufft import NufftPlan, nufft_type1, nufft_type2, prepare_points

    g = golden("nufft")
    plan = NufftPlan(dims=q, m=m)
    geom = prepare_points(plan, g[f"q{q}_m{m}_pts"])
    assert rel(nufft_type1(plan, geom, g[f"q{q}_m{m}_w"]), g[f"q{q}_m{m}_type1"]) <= TOL
    assert rel(nufft_type2(plan, geom, g[f"q{q}_m{m}_c"]), g[f"q{q}_m{m}_type2"]) <= TOL


def test_nufft_windows_and_cutoffs(cuda):
    from paper_2404_17344_b200.nufft import GAUSSIAN_WINDOW, NufftPlan, nufft_type2

    g = golden("nufft")
    out = nufft_type2(NufftPlan(dims=2, m=16, window=GAUSSIAN_WINDOW), g["gw_pts"], g["gw_c"])
    assert rel(out, g["gw_type2"]) <= TOL
    for cutoff in (2, 4, 5, 8):
        assert rel(nufft_type2(NufftPlan(dims=2, m=16, cutoff=cutoff), g["gw_pts"], g["gw_c"]),
                   g[f"cut{cutoff}_type2"]) <= TOL
        assert rel(nufft_type2(NufftPlan(dims=3, m=8, cutoff=cutoff), g["q3cut_pts"], g["q3cut_c"]),
                   g[f"q3cut{cutoff}_type2"]) <= TOL


def test_cross_matvec_matches_reference(cuda):
    from paper_2404_17344_b200.fastsum import build_plan, fast_cross_matvec, prepare_eval_points
    from paper_2404_17344_b200.kernels import KernelSpec
    from paper_2404_17344_b200.windows import WindowSet

    g = golden("cross")
    ws = WindowSet(((1, 2), (3, 4)), d_max=2)
    tr = _ds(g["Xtr"], 2)
    te = _ds(g["Xte"], 2)
    plan = build_plan(KernelSpec("gauss", 1.0 / np.sqrt(2.0)), ws, "default", tr)
    geoms = prepare_eval_points(plan, te)
    out = fast_cross_matvec(plan, geoms, g["v"], 80)
    assert rel(out, g["fast"]) <= TOL
    assert rel(out, g["dense"]) < 1e-3


def test_generic_kernels_agree_with_tiled(cuda):
    """The one-thread-per-point kernels (tuning generic_kernels=1) and the tiled ones."""
    from paper_2404_17344_b200.fastsum import fast_matvec

    for name in ("c2", "c4"):
        g = golden(name)
        tiled = fast_matvec(_plan(g), g["V"][0])
        generic = fast_matvec(_plan(g, tuning={"generic_kernels": 1}), g["V"][0])
        assert rel(tiled, generic) <= 1e-13


def test_native_library_is_what_runs(cuda):
    from paper_2404_17344_b200 import _native
    from paper_2404_17344_b200.fastsum import fast_matvec

    g = golden("c1")
    plan = _plan(g)
    before = _native.launch_count()
    fast_matvec(plan, g["V"][0])
    assert _native.launch_count() > before


@pytest.mark.parametrize("variant", [
    {"weight_tables": 0},                       # weights evaluated per pass (no plan-time table)
    {"cell_items3": 2, "chunk3": 256},          # supercell items, small chunks
    {"cell_items3": 1},                         # single-cell work items (auto-selected for dense data)
    {"cell_items3": 1, "chunk3": 100},
    {"cell_items3": 1, "rhs_pair_spread": 0},   # single-cell hybrid DMMA + DFMA spread for every RHS
    {"cell_items3": 1, "rhs_pair_spread": 0, "tc_spread3": 0},   # ... the register-tiled DFMA spread
    {"cell_items3": 2, "tc_spread3": 0},        # supercell DFMA spread (no 8-RHS tensor-core kernel)
    {"cell_items3": 2, "tc_spread3": 1},        # supercell DFMA spread, single-cell hybrid only
    # split items: supercell spread, single-cell interpolation over the same sorted points
    {"dense_cells3": 1e9, "dense_cells3_interp": 0},
    {"dense_cells3": 1e9, "dense_cells3_interp": 0, "chunk3": 100},
    {"generic_kernels": 1},
    {"sparse_warps": 1},                        # one warp per supercell item (default: two share the tile)
    {"sparse_warps": 1, "cell_items3": 2, "chunk3": 100},
])
def test_kernel_variants_match_reference(cuda, variant):
    """Every plan-time kernel choice (ak_tuning) reproduces the reference."""
    from paper_2404_17344_b200.fastsum import fast_matvecs

    for name in ("c3", "c4"):
        g = golden(name)
        plan = _plan(g, tuning=variant)
        res = fast_matvecs(plan, g["V"], dell="dK_dell_default" in g)
        assert rel(res["K"], g["K_default"]) <= TOL, (variant, name)
        if "dK_dell_default" in g:
            assert rel(res["dK_dell"], g["dK_dell_default"]) <= TOL, (variant, name)


def test_fused_band_transforms_match_cufft(cuda):
    """The band-pruned, multiplier-fused 3-D transform stage (ak_fft3.cuh) against the
    full cuFFT transforms + band multiply (tuning fused_fft3=0) and the reference
    goldens: default and rough presets, K and dK/dl, 8 RHS."""
    from paper_2404_17344_b200.fastsum import fast_matvecs

    cufft = {"fused_fft3": 0}
    for name in ("c3", "c4"):
        g = golden(name)
        dell = "dK_dell_default" in g
        outs = {}
        for mode in ("fused", "cufft"):
            outs[mode] = fast_matvecs(_plan(g, tuning=cufft if mode == "cufft" else None), g["V"], dell=dell)
            assert rel(outs[mode]["K"], g["K_default"]) <= TOL, (mode, name)
        assert rel(outs["fused"]["K"], outs["cufft"]["K"]) <= 1e-13, name
        if dell:
            assert rel(outs["fused"]["dK_dell"], outs["cufft"]["dK_dell"]) <= 1e-13, name
    g = golden("c4")
    for mode in ("fused", "cufft"):
        outs[mode] = fast_matvecs(_plan(g, preset="rough", tuning=cufft if mode == "cufft" else None), g["V"])["K"]
    assert rel(outs["fused"], outs["cufft"]) <= 1e-13


@pytest.mark.parametrize("sc2", ["1", "8"])
def test_q2_item_kernels_match_reference(cuda, sc2):
    """2-D windows through the single-cell tensor-core kernels (tuning cell_items2=1) and
    the lane-per-point kernels (8): configs 2 and 5 and the q = 2 NUFFT goldens."""
    from paper_2404_17344_b200.fastsum import build_mixed_plan, fast_matvecs, mixed_matvecs
    from paper_2404_17344_b200.kernels import KernelSpec
    from paper_2404_17344_b200.nufft import NufftPlan, nufft_type1, nufft_type2, prepare_points

    tun = {"cell_items2": int(sc2)}
    g = golden("c2")
    res = fast_matvecs(_plan(g, tuning=tun), g["V"], dell=True)
    assert rel(res["K"], g["K_default"]) <= TOL
    assert rel(res["dK_dell"], g["dK_dell_default"]) <= TOL
    g = golden("c5")
    specs = [KernelSpec(str(f), float(l), 1.0) for f, l in zip(g["families"], g["ells"])]
    res = mixed_matvecs(build_mixed_plan(specs, _ws(g), "default", _ds(g["X"], g["d_max"]), tuning=tun), g["V"])
    assert rel(res["K"], g["K_default"]) <= TOL
    for w in range(len(specs)):
        assert rel(res["dK_dell"][w], g["dK_dell_default"][w]) <= TOL
    g = golden("nufft")
    for m in (8, 16):
        plan = NufftPlan(dims=2, m=m)
        geom = prepare_points(plan, g[f"q2_m{m}_pts"], tuning=tun)
        assert rel(nufft_type1(plan, geom, g[f"q2_m{m}_w"]), g[f"q2_m{m}_type1"]) <= TOL
        assert rel(nufft_type2(plan, geom, g[f"q2_m{m}_c"]), g[f"q2_m{m}_type2"]) <= TOL


def test_plan_options_match_reference(cuda):
    """build_plan(cutoff, oversampling, window, explicit m) on mixed window lengths, and the
    dense-cell regime (single-cell tensor-core items) for all four families."""
    from paper_2404_17344_b200.fastsum import build_plan, fast_matvec
    from paper_2404_17344_b200.kernels import KernelSpec
    from paper_2404_17344_b200.windows import WindowSet

    g = golden("plan_options")
    ws = WindowSet(((1, 2, 3), (4, 5), (6,)), d_max=3)
    ds = _ds(g["X"], 3)
    opts = {"cut3": dict(cutoff=3), "cut4": dict(cutoff=4), "cut5": dict(cutoff=5), "cut8": dict(cutoff=8),
            "os1p5": dict(oversampling=1.5), "os3": dict(oversampling=3.0),
            "gaussw": dict(window="gaussian_window"), "gaussw_cut4": dict(window="gaussian_window", cutoff=4)}
    for fam in ("gauss", "matern12"):
        spec = KernelSpec(fam, 0.35, 0.8)
        for key, kw in opts.items():
            assert rel(fast_matvec(build_plan(spec, ws, "default", ds, **kw), g["v"]), g[f"{fam}_{key}"]) <= TOL, key
        assert rel(fast_matvec(build_plan(spec, ws, 24, ds), g["v"]), g[f"{fam}_m24"]) <= TOL
    dsd = _ds(g["Xd"], 3)
    for fam in ("gauss", "der_gauss", "matern12", "der_matern12"):
        plan = build_plan(KernelSpec(fam, 0.3, 1.0), ws, "default", dsd)
        assert rel(fast_matvec(plan, g["vd"]), g[f"dense_{fam}"]) <= TOL, fam


def test_nufft_dense_boundary_cells(cuda):
    """Densely occupied cells on the periodic boundary: single-cell items, wrapping footprints."""
    from paper_2404_17344_b200.nufft import NufftPlan, nufft_type1, nufft_type2, prepare_points

    g = golden("nufft_dense")
    for q in (2, 3):
        plan = NufftPlan(dims=q, m=32)
        geom = prepare_points(plan, g[f"q{q}_pts"])
        assert rel(nufft_type1(plan, geom, g[f"q{q}_w"]), g[f"q{q}_type1"]) <= TOL
        assert rel(nufft_type2(plan, geom, g[f"q{q}_c"]), g[f"q{q}_type2"]) <= TOL


@pytest.mark.parametrize("cutoff", [5, 6])
def test_dense_cells_cutoff(cuda, cutoff):
    """Densely occupied cells (single-cell kernels) at cutoff 5 -- a 10-tap window padded to
    the 12-tap kernels, whose lane tiles then skip the zero taps -- and at the default 6,
    against the oracle with the same cutoff."""
    from oracle import restate as R
    from paper_2404_17344_b200.fastsum import build_plan, fast_matvecs
    from paper_2404_17344_b200.kernels import KernelSpec
    from paper_2404_17344_b200.windows import WindowSet

    rng = np.random.default_rng(31)
    X = rng.uniform(-0.01, 0.01, size=(4000, 6))
    V = rng.normal(size=(2, 4000))
    ws = WindowSet(((1, 2, 3), (4, 5, 6)), d_max=3)
    plan = build_plan(KernelSpec("gauss", 0.3), ws, "default", _ds(X, 3), cutoff=cutoff)
    res = fast_matvecs(plan, V, dell=True)
    for fam, key in (("gauss", "K"), ("der_gauss", "dK_dell")):
        fs = R.FastSum(fam, 0.3, 1.0, [(0, 1, 2), (3, 4, 5)], X, cutoff=cutoff)
        for r in range(2):
            assert rel(res[key][r], fs.matvec(V[r])) <= TOL, (cutoff, key, r)


@pytest.mark.parametrize("layout", ["corner", "wrap", "full", "two_boxes"])
def test_occupied_box_transforms_match_full(cuda, layout):
    """The fused 3-D transforms work on each window's occupied grid box (ak_geom_box):
    data in a corner, data straddling the periodic seam on one axis (a box that wraps
    around n), data over the whole torus (full box) and two windows with different
    boxes, against the whole-grid cuFFT stage (fused_fft3=0): K and dK/dl, 3 RHS, plus a
    cross product whose evaluation points sit in another box than the training points."""
    from paper_2404_17344_b200.fastsum import (build_plan, fast_cross_matvec, fast_matvecs,
                                               prepare_eval_points)
    from paper_2404_17344_b200.kernels import KernelSpec
    from paper_2404_17344_b200.windows import WindowSet

    rng = np.random.default_rng(7)
    N = 3000

    def pts(kind, n):
        if kind == "corner":
            return rng.uniform(-0.12, 0.03, size=(n, 3))
        if kind == "wrap":
            X = rng.uniform(-0.1, 0.1, size=(n, 3))
            X[:, 0] = np.where(rng.random(n) < 0.5, rng.uniform(0.43, 0.5, n), rng.uniform(-0.5, -0.44, n))
            return X
        return rng.uniform(-0.5, 0.5, size=(n, 3))

    if layout == "two_boxes":
        X = np.hstack([pts("corner", N), pts("wrap", N)])
        ws = WindowSet(((1, 2, 3), (4, 5, 6)), d_max=3)
    else:
        X = pts(layout, N)
        ws = WindowSet(((1, 2, 3),), d_max=3)
    X = np.minimum(X, 0.5 - 1e-12)
    spec = KernelSpec("gauss", 0.3)
    V = rng.normal(size=(3, N))
    fused = build_plan(spec, ws, "default", _ds(X, 3))
    ref = build_plan(spec, ws, "default", _ds(X, 3), tuning={"fused_fft3": 0})
    boxes = fused.geometries.boxes
    n = fused.geometries.n
    if layout == "corner":
        assert all(L < n for _, L in boxes[0])
    if layout == "wrap":
        lo, L = boxes[0][0]
        assert L < n and lo + L > n  # wraps around the seam
    if layout == "full":
        assert boxes[0] == ((0, n),) * 3
    a = fast_matvecs(fused, V, dell=True)
    b = fast_matvecs(ref, V, dell=True)
    assert rel(a["K"], b["K"]) <= 1e-13
    assert rel(a["dK_dell"], b["dK_dell"]) <= 1e-13
    Xe = np.minimum(pts("full" if layout == "corner" else "corner", 500), 0.5 - 1e-12)
    if layout == "two_boxes":
        Xe = np.hstack([Xe, pts("corner", 500)])
    v = V[0]
    ca = fast_cross_matvec(fused, prepare_eval_points(fused, _ds(Xe, 3)), v, 500)
    cb = fast_cross_matvec(ref, prepare_eval_points(ref, _ds(Xe, 3)), v, 500)
    assert rel(ca, cb) <= 1e-13
