"""Pin the CPU oracle (oracle/) against the reference's own golden vectors
(tests/golden/, produced by the reference by make_golden.py) and against the
reference test suite's known answers.  CPU only."""

import math

import numpy as np
import pytest

from conftest import golden, rel, windows_of
from oracle import restate as R


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4"])
def test_oracle_matches_reference_configs(name):
    g = golden(name)
    fam = str(g["families"][0])
    ell = float(g["ells"][0])
    sf = float(g["sigma_f"])
    wins = windows_of(g)
    fs = R.FastSum(fam, ell, sf, wins, g["X"])
    for r, v in enumerate(g["V"]):
        assert rel(fs.matvec(v), g["K_default"][r]) <= 1e-14
    if "dK_dell_default" in g:
        dfs = R.FastSum("der_" + fam, ell, sf, wins, g["X"])
        for r, v in enumerate(g["V"]):
            assert rel(dfs.matvec(v), g["dK_dell_default"][r]) <= 1e-14
    if "K_dense" in g:
        for r, v in enumerate(g["V"]):
            assert rel(R.dense_matvec(fam, ell, sf, wins, g["X"], v), g["K_dense"][r]) <= 1e-13


def test_oracle_matches_reference_mixed_c5():
    g = golden("c5")
    wins = windows_of(g)
    for r, v in enumerate(g["V"]):
        acc = np.zeros_like(v)
        for k, w in enumerate(wins):
            fs = R.FastSum(str(g["families"][k]), float(g["ells"][k]), 1.0, [w], g["X"])
            acc += fs.matvec(v)
            d = R.FastSum("der_" + str(g["families"][k]), float(g["ells"][k]), 1.0, [w], g["X"]).matvec(v)
            assert rel(d, g["dK_dell_default"][k, r]) <= 1e-14
        assert rel(acc, g["K_default"][r]) <= 1e-14


def test_oracle_presets():
    g = golden("c1_presets")
    wins = windows_of(g)
    for preset in ("rough", "fine"):
        fs = R.FastSum("gauss", float(g["ells"][0]), 1.0, wins, g["X"], m=R.PRESETS[preset])
        assert rel(fs.matvec(g["V"][0]), g[f"K_{preset}"][0]) <= 1e-14


def test_oracle_family_grid():
    g = golden("family_grid")
    for fam in ("gauss", "der_gauss", "matern12", "der_matern12"):
        for ell in (0.1, 1.0, 10.0):
            for preset in ("rough", "default", "fine"):
                fs = R.FastSum(fam, ell, math.sqrt(0.5), [(0, 1, 2), (3, 4, 5)], g["X"], m=R.PRESETS[preset])
                assert rel(fs.matvec(g["v"]), g[f"{fam}_{ell}_{preset}"]) <= 1e-13


@pytest.mark.parametrize("q", [1, 2, 3])
@pytest.mark.parametrize("m", [8, 16])
def test_oracle_nufft_golden(q, m):
    g = golden("nufft")
    plan = R.Nufft(q, m)
    geom = R.Geometry(plan, g[f"q{q}_m{m}_pts"])
    assert rel(R.type1(plan, geom, g[f"q{q}_m{m}_w"]), g[f"q{q}_m{m}_type1"]) <= 1e-14
    assert rel(R.type2(plan, geom, g[f"q{q}_m{m}_c"]), g[f"q{q}_m{m}_type2"]) <= 1e-14


def test_oracle_nufft_windows_and_cutoffs():
    g = golden("nufft")
    plan = R.Nufft(2, 16, window="gaussian_window")
    assert rel(R.type2(plan, R.Geometry(plan, g["gw_pts"]), g["gw_c"]), g["gw_type2"]) <= 1e-14
    for cutoff in (2, 4, 5, 8):
        plan = R.Nufft(2, 16, cutoff=cutoff)
        assert rel(R.type2(plan, R.Geometry(plan, g["gw_pts"]), g["gw_c"]), g[f"cut{cutoff}_type2"]) <= 1e-14
        plan3 = R.Nufft(3, 8, cutoff=cutoff)
        out = R.type2(plan3, R.Geometry(plan3, g["q3cut_pts"]), g["q3cut_c"])
        assert rel(out, g[f"q3cut{cutoff}_type2"]) <= 1e-14


@pytest.mark.parametrize("q", [1, 2, 3])
def test_oracle_type1_type2_vs_direct(q):
    """Reference test_nufft.py:112-146 known answers, at the same 1e-8 bar."""
    m = 8
    plan = R.Nufft(q, m)
    rng = np.random.default_rng(q)
    pts = rng.uniform(-0.5, 0.4999, size=(10, q))
    c = rng.normal(size=(m,) * q) + 1j * rng.normal(size=(m,) * q)
    w = rng.normal(size=10) + 1j * rng.normal(size=10)
    geom = R.Geometry(plan, pts)
    ref2 = R.direct_type2(m, q, pts, c)
    assert np.max(np.abs(R.type2(plan, geom, c) - ref2)) / np.max(np.abs(ref2)) <= 1e-8
    ref1 = R.direct_type1(m, q, pts, w)
    assert np.max(np.abs(R.type1(plan, geom, w) - ref1)) / np.max(np.abs(ref1)) <= 1e-8


def test_oracle_dense_known_answer():
    """Single point: K v = sigma_f^2 * P * v (reference test_kernels.py:46-51)."""
    X = np.array([[0.01, -0.02, 0.03, 0.0, 0.1, -0.1]])
    out = R.dense_matvec("gauss", 1.0, 2.0, [(0, 1, 2), (3, 4, 5)], X, np.array([3.0]))
    assert abs(out[0] - 4.0 * 2 * 3.0) < 1e-12


def test_oracle_cg_matches_reference_krr():
    """krr_fit (solver.py:99-120) restated: same CG iterations, same coefficients."""
    g = golden("solver")
    sf = math.sqrt(1 / 3)
    fs = R.FastSum("gauss", 0.6 / math.sqrt(2), sf, [(0, 1), (2, 3), (4, 5)], g["Xtr"])
    x, it = R.cg_solve(fs.matvec, g["ytr"], 0.05)
    assert it == int(g["iters"])
    assert rel(x, g["coef"]) <= 1e-10


def test_oracle_gsi_matches_reference():
    """compute_gsi (gsi.py:72-102) restated on the oracle's type-1 transforms."""
    from itertools import product

    g = golden("solver")
    gg = golden("gsi")
    sf = math.sqrt(1 / 3)
    wins = [(0, 1), (2, 3), (4, 5)]
    fs = R.FastSum("gauss", 0.6 / math.sqrt(2), sf, wins, g["Xtr"])
    thetas = {}
    nz = R.freqs(32) != 0
    for k, w in enumerate(wins):
        S = np.conj(R.type1(fs.plans[2], fs.geoms[k], g["coef"]))
        power = np.abs(fs.tables[2] * S) ** 2
        for pat in product((0, 1), repeat=2):
            if not any(pat):
                continue
            mask = (nz if pat[0] else ~nz)[:, None] & (nz if pat[1] else ~nz)[None, :]
            key = ",".join(str(w[a] + 1) for a in range(2) if pat[a])
            thetas[key] = thetas.get(key, 0.0) + float(power[mask].sum())
    got = np.array([thetas[k] for k in gg["keys"]])
    assert rel(got, gg["thetas"]) <= 1e-12


def test_chunked_oracle_equals_plain():
    """The bench reference arm's row-chunked, thread-pooled product equals the plain oracle."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import restate as R

    rng = np.random.default_rng(11)
    X = rng.uniform(-0.14, 0.14, size=(700, 6))
    v = rng.normal(size=700)
    windows = [(0, 1, 2), (3, 4), (5,)]
    plain = R.FastSum("gauss", 0.3, 1.0, windows, X).matvec(v)
    chunked = R.ChunkedFastSum("gauss", 0.3, 1.0, windows, X, chunks=3)
    with ThreadPoolExecutor(4) as pool:
        out = chunked.matvec_pool(v, pool)
    assert np.linalg.norm(out - plain) <= 1e-13 * np.linalg.norm(plain)


def test_oracle_plan_options_match_reference():
    """cutoff / oversampling / Gaussian window / explicit m, and densely occupied cells."""
    from oracle import restate as R

    g = golden("plan_options")
    wins = [(0, 1, 2), (3, 4), (5,)]
    opts = {"cut3": dict(cutoff=3), "cut4": dict(cutoff=4), "cut5": dict(cutoff=5), "cut8": dict(cutoff=8),
            "os1p5": dict(oversampling=1.5), "os3": dict(oversampling=3.0),
            "gaussw": dict(window="gaussian_window"), "gaussw_cut4": dict(window="gaussian_window", cutoff=4)}
    for fam in ("gauss", "matern12"):
        for key, kw in opts.items():
            out = R.FastSum(fam, 0.35, 0.8, wins, g["X"], **kw).matvec(g["v"])
            assert rel(out, g[f"{fam}_{key}"]) <= 1e-13, (fam, key)
        assert rel(R.FastSum(fam, 0.35, 0.8, wins, g["X"], m=24).matvec(g["v"]), g[f"{fam}_m24"]) <= 1e-13
    for fam in ("gauss", "der_gauss", "matern12", "der_matern12"):
        out = R.FastSum(fam, 0.3, 1.0, wins, g["Xd"]).matvec(g["vd"])
        assert rel(out, g[f"dense_{fam}"]) <= 1e-13, fam


def test_oracle_nufft_dense_boundary_cells():
    from oracle import restate as R

    g = golden("nufft_dense")
    for q in (2, 3):
        plan = R.Nufft(q, 32)
        geom = R.Geometry(plan, g[f"q{q}_pts"])
        assert rel(R.type1(plan, geom, g[f"q{q}_w"]), g[f"q{q}_type1"]) <= 1e-13
        assert rel(R.type2(plan, geom, g[f"q{q}_c"]), g[f"q{q}_type2"]) <= 1e-13


def test_fullsize_oracle_matches_reference_c5_and_c3():
    """oracle/fullsize.py (row chunks on a thread pool, one window at a time, one
    spread shared by K and dK/dl) reproduces the reference's own outputs."""
    from oracle.fullsize import products

    g = golden("c5")
    wins = windows_of(g)
    specs = [(str(g["families"][k]), float(g["ells"][k]), 1.0) for k in range(len(wins))]
    res = products(g["X"], wins, specs, g["V"], dell=True, per_window_dell=True, threads=4, chunks=3)
    for r in range(len(g["V"])):
        assert rel(res["K"][r], g["K_default"][r]) <= 1e-13
        for k in range(len(wins)):
            assert rel(res["dK_dell"][k, r], g["dK_dell_default"][k, r]) <= 1e-13
    g = golden("c3")
    fam, ell, sf = str(g["families"][0]), float(g["ells"][0]), float(g["sigma_f"])
    wins = windows_of(g)
    res = products(g["X"], wins, [(fam, ell, sf)] * len(wins), g["V"], dell=True, threads=3, chunks=5)
    for r in range(len(g["V"])):
        assert rel(res["K"][r], g["K_default"][r]) <= 1e-13
        assert rel(res["dK_dell"][r], g["dK_dell_default"][r]) <= 1e-13


def test_bounds_match_reference():
    """oracle/bounds.py (Theorems 3.2/3.3) reproduces the reference's analytic_bound
    (bounds.py:103-130) on a grid covering every branch, including eta < 1 refusals,
    and dominates the reference's measured worst case."""
    from oracle import bounds as B

    g = golden("bounds")
    for fam in ("gauss", "der_gauss"):
        for q in (1, 3):
            tab = g[f"{fam}_q{q}"]
            for i, ell in enumerate(g["ells"]):
                for j, m in enumerate(g["ms"]):
                    if np.isnan(tab[i, j]):
                        with pytest.raises(B.EtaTooSmall):
                            B.analytic_bound(fam, q, float(ell), int(m))
                    else:
                        got = B.analytic_bound(fam, q, float(ell), int(m))
                        assert abs(got - tab[i, j]) <= 1e-14 * abs(tab[i, j]), (fam, q, ell, m)
    cells = (("gauss", 1, 0.1, 16), ("gauss", 3, 0.3, 16), ("der_gauss", 1, 0.2, 16), ("der_gauss", 3, 0.5, 8))
    for (fam, q, ell, m), meas in zip(cells, g["measured"]):
        assert meas <= B.analytic_bound(fam, q, ell, m)
    with pytest.raises(ValueError):
        B.analytic_bound("matern12", 3, 1.0, 32)
    with pytest.raises(ValueError):
        B.analytic_bound("gauss", 2, 1.0, 32)


def test_oracle_c1_within_paper_bound():
    """The reference algorithm (oracle) on BASELINE config 1 at full size stays within the
    per-entry analytic bound of the exact dense product."""
    from oracle.bounds import per_entry_bound

    from paper_2404_17344_b200 import configs

    wl = configs.config1()
    cols = [wl.window_set.columns(w) for w in wl.window_set]
    v = wl.V[0]
    for fam in ("gauss", "der_gauss"):
        fast = R.FastSum(fam, wl.spec.ell, 1.0, cols, wl.data.features).matvec(v)
        dense = R.dense_matvec(fam, wl.spec.ell, 1.0, cols, wl.data.features, v)
        bound = per_entry_bound(fam, wl.window_set.lengths, wl.spec.ell, 32, 1.0, v)
        assert np.max(np.abs(fast - dense)) <= bound
