"""GPU: seeded random configurations against the CPU oracle (robustness sweep).

Each case draws N (1 .. 20k, log-uniform), 1-4 windows of length 1-3 over 6
features, a preset or explicit m, a kernel family, a node distribution
(uniform box, clustered, hugging the periodic boundary, all in one cell), R
right-hand sides and plan knobs (supercell edge, item cap), and checks K V
(and dK/dl V for base families) against the oracle at the north_star
tolerance.  The cases are fixed by their seeds, so failures reproduce."""

import math
import os

import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu

TOL = 1e-8
N_CASES = int(os.environ.get("AK_FUZZ_CASES", "64"))   # a longer campaign: AK_FUZZ_CASES=600


def _case(seed):
    rng = np.random.default_rng(10_000 + seed)
    lo = 0.0 if rng.random() < 0.25 else math.log(100)
    N = int(round(math.exp(rng.uniform(lo, math.log(20_000)))))
    P = int(rng.integers(1, 5))
    windows = []
    for _ in range(P):
        q = int(rng.integers(1, 4))
        w = tuple(sorted(int(c) for c in rng.choice(6, size=q, replace=False)))
        if w not in windows:
            windows.append(w)
    preset = rng.choice(["rough", "default", "fine", "explicit"])
    if preset == "explicit":
        preset = int(rng.integers(4, 25)) * 2
    family = str(rng.choice(["gauss", "der_gauss", "matern12", "der_matern12"]))
    ell = float(math.exp(rng.uniform(math.log(0.05), math.log(3.0))))
    dist = rng.choice(["uniform", "cluster", "boundary", "onecell"])
    if dist == "uniform":
        X = rng.uniform(-0.25, 0.25, size=(N, 6)) / math.sqrt(3.0)
    elif dist == "cluster":
        X = np.clip(rng.normal(scale=0.02, size=(N, 6)) + rng.uniform(-0.1, 0.1, size=(1, 6)), -0.49, 0.49)
    elif dist == "boundary":
        X = np.where(rng.random((N, 6)) < 0.5, rng.uniform(-0.5, -0.47, (N, 6)), rng.uniform(0.47, 0.5, (N, 6)))
        X = np.minimum(X, np.nextafter(0.5, 0.0))
    else:
        X = 0.003 + 1e-4 * rng.random((N, 6))
    R = int(rng.choice([1, 2, 5, 8, 9, 16]))   # 9: the RHS-batched q <= 2 kernels; 8, 16: RHS chunks of 8 (sparse 3-D spread)
    V = rng.normal(size=(R, N))
    knobs = {}
    k = rng.integers(0, 4)
    if k == 1:
        knobs["cell_items3"] = 1
    elif k == 2:
        knobs["cell_items3"] = 2
    elif k == 3:
        knobs["dense_cells3"] = 1e9
        knobs["dense_cells3_interp"] = 0.0
    if rng.random() < 0.3:
        knobs["chunk3"] = int(rng.choice([64, 100, 333]))
    masks = None
    if rng.random() < 0.25:   # row-masked windows (the cell-slab layout's plans)
        masks = rng.random((len(windows), N)) < rng.uniform(0.2, 1.0, size=(len(windows), 1))
    return dict(N=N, windows=windows, preset=preset, family=family, ell=ell, dist=str(dist), X=X, V=V,
                knobs=knobs, masks=masks)


@pytest.mark.parametrize("seed", range(N_CASES))
def test_random_configuration_matches_oracle(cuda, seed):
    from oracle import restate as R
    from paper_2404_17344_b200.dataset import PRESCALED, Dataset
    from paper_2404_17344_b200.fastsum import PRESETS, build_plan, fast_matvecs
    from paper_2404_17344_b200.kernels import DERIVATIVE_PREFACTOR, KernelSpec
    from paper_2404_17344_b200.windows import WindowSet

    c = _case(seed)
    ds = Dataset(c["X"], np.zeros(c["N"]), tuple(f"x{i}" for i in range(6)), scaling_state=PRESCALED, d_max=3)
    ws = WindowSet(tuple(tuple(col + 1 for col in w) for w in c["windows"]), d_max=3)
    spec = KernelSpec(c["family"], c["ell"], 0.7)
    import warnings

    with warnings.catch_warnings():
        warnings.simplefilter("ignore")  # AccuracyWarning for small ell * m is expected here
        plan = build_plan(spec, ws, c["preset"], ds, row_masks=c["masks"], tuning=c["knobs"])
    base = DERIVATIVE_PREFACTOR[c["family"]] is None
    res = fast_matvecs(plan, c["V"], dell=base)
    m = PRESETS.get(c["preset"], c["preset"])

    def oracle(family, v):
        if c["masks"] is None:
            return R.FastSum(family, c["ell"], 0.7, c["windows"], c["X"], m=m).matvec(v)
        out = np.zeros(c["N"])
        for w, mask in zip(c["windows"], c["masks"]):
            rows = np.flatnonzero(mask)
            if len(rows):
                out[rows] += R.FastSum(family, c["ell"], 0.7, [w], c["X"][rows], m=m).matvec(v[rows])
        return out

    for r in range(c["V"].shape[0]):
        ref = oracle(c["family"], c["V"][r])
        if not np.any(ref):
            assert not np.any(res["K"][r]), (seed, "masked-empty")
            continue
        assert rel(res["K"][r], ref) <= TOL, (seed, c["dist"], c["knobs"], r, c["masks"] is not None)
    if base:
        ref = oracle("der_" + c["family"], c["V"][0])
        if np.any(ref):
            assert rel(res["dK_dell"][0], ref) <= TOL, (seed, "dK")


@pytest.mark.parametrize("seed", range(16))
def test_random_nufft_matches_oracle(cuda, seed):
    """Type-1 / type-2 NUFFTs: random q, m (even, 2..64), N (0..5000), node distribution."""
    from oracle import restate as R
    from paper_2404_17344_b200.nufft import NufftPlan, nufft_type1, nufft_type2, prepare_points

    rng = np.random.default_rng(20_000 + seed)
    q = int(rng.integers(1, 4))
    m = int(rng.integers(1, 33)) * 2 if q < 3 else int(rng.integers(1, 17)) * 2
    N = int(rng.integers(0, 5001))
    if rng.random() < 0.5:
        pts = rng.uniform(-0.5, 0.5, size=(N, q))
    else:
        pts = np.clip(rng.normal(scale=0.01, size=(N, q)) + rng.uniform(-0.5, 0.5, size=(1, q)), -0.5, 0.4999)
    pts = np.minimum(pts, np.nextafter(0.5, 0.0))
    w = rng.normal(size=N) + 1j * rng.normal(size=N)
    c = rng.normal(size=(m,) * q) + 1j * rng.normal(size=(m,) * q)
    plan = NufftPlan(dims=q, m=m)
    oplan = R.Nufft(q, m)
    if N == 0:
        assert np.all(nufft_type1(plan, pts, w) == 0)
        return
    geom = prepare_points(plan, pts)
    ogeom = R.Geometry(oplan, pts)
    assert rel(nufft_type1(plan, geom, w), R.type1(oplan, ogeom, w)) <= TOL, (seed, q, m, N)
    assert rel(nufft_type2(plan, geom, c), R.type2(oplan, ogeom, c)) <= TOL, (seed, q, m, N)


@pytest.mark.parametrize("seed", range(12))
def test_random_cross_matvec_matches_oracle(cuda, seed):
    """K(eval, train) v with train / eval sets of different size and density (their own
    item lists: the eval geometry may pick other supercell edges than the train one)."""
    from oracle import restate as R
    from paper_2404_17344_b200.dataset import PRESCALED, Dataset
    from paper_2404_17344_b200.fastsum import build_plan, fast_cross_matvec, prepare_eval_points
    from paper_2404_17344_b200.kernels import KernelSpec
    from paper_2404_17344_b200.windows import WindowSet

    rng = np.random.default_rng(30_000 + seed)
    windows = [(0, 1, 2), (3, 4)] if seed % 2 else [(0, 1, 2), (2, 3, 4), (5,)]
    Ntr = int(rng.integers(50, 20000))
    Nte = int(rng.integers(1, 20000))
    spread_tr = float(rng.choice([0.01, 0.05, 0.14]))
    spread_te = float(rng.choice([0.01, 0.05, 0.14]))
    Xtr = rng.uniform(-spread_tr, spread_tr, size=(Ntr, 6))
    Xte = rng.uniform(-spread_te, spread_te, size=(Nte, 6))
    v = rng.normal(size=Ntr)
    fam = str(rng.choice(["gauss", "matern12", "der_gauss"]))
    ell = float(rng.uniform(0.1, 1.0))

    def ds(X):
        return Dataset(X, np.zeros(X.shape[0]), tuple(f"x{i}" for i in range(6)), scaling_state=PRESCALED, d_max=3)

    plan = build_plan(KernelSpec(fam, ell, 0.8), WindowSet(tuple(tuple(c + 1 for c in w) for w in windows), d_max=3),
                      "default", ds(Xtr))
    out = fast_cross_matvec(plan, prepare_eval_points(plan, ds(Xte)), v, Nte)
    # oracle composition of fastsum.py:180-191: spread at train, interp at eval, per window
    acc = np.zeros(Nte, dtype=np.complex128)
    for w in windows:
        nplan = R.Nufft(len(w), 32)
        S = R.type1(nplan, R.Geometry(nplan, Xtr[:, list(w)]), v)
        acc += R.type2(nplan, R.Geometry(nplan, Xte[:, list(w)]), R.kernel_coefficients(fam, ell, len(w), 32) * S)
    ref = R.operator_scale(fam, ell, 0.8) * acc.real
    assert rel(out, ref) <= TOL, (seed, Ntr, Nte, spread_tr, spread_te)


@pytest.mark.parametrize("seed", range(8))
def test_random_mixed_plan_matches_oracle(cuda, seed):
    """Per-window family and length-scale (MixedKernelPlan): K V, the per-window dK/dl_w V
    and dK/dsigma_f V against sums of single-window oracle products."""
    from oracle import restate as R
    from paper_2404_17344_b200.dataset import PRESCALED, Dataset
    from paper_2404_17344_b200.fastsum import build_mixed_plan, mixed_matvecs
    from paper_2404_17344_b200.kernels import KernelSpec
    from paper_2404_17344_b200.windows import WindowSet

    rng = np.random.default_rng(40_000 + seed)
    P = int(rng.integers(2, 6))
    windows = []
    while len(windows) < P:
        q = int(rng.integers(1, 4))
        w = tuple(sorted(int(c) for c in rng.choice(7, size=q, replace=False)))
        if w not in windows:
            windows.append(w)
    N = int(rng.integers(100, 8000))
    X = np.clip(rng.normal(scale=float(rng.choice([0.01, 0.05])), size=(N, 7)), -0.49, 0.49)
    R_ = int(rng.choice([1, 3]))
    V = rng.normal(size=(R_, N))
    fams = [str(rng.choice(["gauss", "matern12"])) for _ in windows]
    ells = [float(rng.uniform(0.1, 1.5)) for _ in windows]
    sf = 0.9
    ds = Dataset(X, np.zeros(N), tuple(f"x{i}" for i in range(7)), scaling_state=PRESCALED, d_max=3)
    specs = [KernelSpec(f, l, sf) for f, l in zip(fams, ells)]
    plan = build_mixed_plan(specs, WindowSet(tuple(tuple(c + 1 for c in w) for w in windows), d_max=3), "default", ds)
    res = mixed_matvecs(plan, V)
    for r in range(R_):
        K = np.zeros(N)
        for w, (win, f, l) in enumerate(zip(windows, fams, ells)):
            Kw = R.FastSum(f, l, sf, [win], X).matvec(V[r])
            dKw = R.FastSum("der_" + f, l, sf, [win], X).matvec(V[r])
            K += Kw
            assert rel(res["dK_dell"][w][r], dKw) <= TOL, (seed, w, r)
        assert rel(res["K"][r], K) <= TOL, (seed, r)
        assert rel(res["dK_dsigma"][r], (2.0 / sf) * K) <= TOL, (seed, r)
