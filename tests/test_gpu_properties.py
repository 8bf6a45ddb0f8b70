"""GPU properties at full BASELINE sizes and edge cases (size-independent
checks: linearity, symmetry, exact rescales, zero input), plus parity against
the CPU oracle where the oracle finishes in seconds."""

import math

import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu


def _ds(X, d_max):
    from paper_2404_17344_b200.dataset import PRESCALED, Dataset

    return Dataset(X, np.zeros(X.shape[0]), tuple(f"x{i + 1}" for i in range(X.shape[1])),
                   scaling_state=PRESCALED, d_max=d_max)


@pytest.fixture(scope="module")
def c4_plan(cuda):
    from paper_2404_17344_b200 import configs
    from paper_2404_17344_b200.fastsum import build_plan

    wl = configs.config4()
    return wl, build_plan(wl.spec, wl.window_set, "default", wl.data)


def test_c4_full_linearity_symmetry_zero(c4_plan):
    from paper_2404_17344_b200.fastsum import fast_dsigma_matvec, fast_matvec

    wl, plan = c4_plan
    N = wl.data.n_rows
    rng = np.random.default_rng(5)
    v, w = rng.normal(size=N), rng.normal(size=N)
    Kv, Kw = fast_matvec(plan, v), fast_matvec(plan, w)
    combo = fast_matvec(plan, 1.5 * v - 2.0 * w)
    assert np.max(np.abs(combo - (1.5 * Kv - 2.0 * Kw))) <= 1e-10 * np.max(np.abs(Kv))
    assert abs(Kv @ w - v @ Kw) <= 1e-8 * np.linalg.norm(v) * np.linalg.norm(w)
    np.testing.assert_array_equal(fast_matvec(plan, np.zeros(N)), np.zeros(N))
    np.testing.assert_allclose(fast_dsigma_matvec(plan, v), 2.0 * Kv, rtol=0, atol=1e-13 * np.max(np.abs(Kv)))


def test_batched_rhs_equal_single(c4_plan):
    from paper_2404_17344_b200.fastsum import fast_matvec, fast_matvecs

    wl, plan = c4_plan
    rng = np.random.default_rng(9)
    V = rng.normal(size=(3, wl.data.n_rows))
    res = fast_matvecs(plan, V, dell=True, dsigma=True)
    for r in range(3):
        assert rel(res["K"][r], fast_matvec(plan, V[r])) <= 1e-13
    assert res["dK_dell"].shape == V.shape
    assert rel(res["dK_dsigma"], 2.0 * res["K"]) <= 1e-15


def test_device_tensors_stay_on_device(c4_plan, cuda):
    from paper_2404_17344_b200.fastsum import fast_matvec

    wl, plan = c4_plan
    v = cuda.as_tensor(wl.V[0], device="cuda")
    out = fast_matvec(plan, v)
    assert out.is_cuda and out.dtype == cuda.float64
    assert rel(out.cpu().numpy(), fast_matvec(plan, wl.V[0])) <= 1e-14


def test_pinned_host_input(c4_plan, cuda):
    """A page-locked caller buffer takes the non-blocking upload; reusing and
    overwriting it between calls must not leak into earlier results."""
    from paper_2404_17344_b200.fastsum import fast_matvec, fast_matvecs

    wl, plan = c4_plan
    buf = cuda.empty(wl.data.n_rows, dtype=cuda.float64, pin_memory=True).numpy()
    buf[:] = wl.V[0]
    first = fast_matvec(plan, buf)
    buf[:] = -wl.V[0]
    second = fast_matvec(plan, buf)
    ref = fast_matvec(plan, np.array(wl.V[0]))
    assert rel(first, ref) <= 1e-14
    assert rel(second, -ref) <= 1e-14
    B = cuda.empty((2, wl.data.n_rows), dtype=cuda.float64, pin_memory=True).numpy()
    B[0], B[1] = wl.V[0], 2.0 * wl.V[0]
    res = fast_matvecs(plan, B)["K"]
    assert rel(res[1], 2.0 * ref) <= 1e-13


def _oracle_check(X, windows, v, family="gauss", ell=0.3, d_max=3, preset="default", sf=1.0, tol=1e-8, tuning=None):
    from oracle import restate as R
    from paper_2404_17344_b200.fastsum import PRESETS, build_plan, fast_matvec
    from paper_2404_17344_b200.kernels import KernelSpec
    from paper_2404_17344_b200.windows import WindowSet

    ws = WindowSet(tuple(tuple(c + 1 for c in w) for w in windows), d_max=d_max)
    plan = build_plan(KernelSpec(family, ell, sf), ws, preset, _ds(X, d_max), tuning=tuning)
    out = fast_matvec(plan, v)
    ref = R.FastSum(family, ell, sf, windows, X, m=PRESETS.get(preset, preset)).matvec(v)
    assert rel(out, ref) <= tol
    return out, ref


def test_single_point(cuda):
    X = np.array([[0.01, -0.02, 0.03]])
    out, ref = _oracle_check(X, [(0, 1, 2)], np.array([2.5]))
    assert out.shape == (1,)


@pytest.mark.parametrize("items", ["auto", "single_cell"])
def test_points_on_the_box_boundary_and_wraparound(cuda, items):
    """Nodes at -1/2, just below +1/2 and on cell boundaries: footprints wrap."""
    tun = {"cell_items2": 1, "cell_items3": 1} if items == "single_cell" else None
    rng = np.random.default_rng(1)
    X = rng.uniform(-0.5, 0.5, size=(600, 6))
    X[:50] = -0.5
    X[50:100] = np.nextafter(0.5, 0.0)
    X[100:150] = np.floor(X[100:150] * 64) / 64  # exact cell boundaries (t integer)
    _oracle_check(X, [(0, 1, 2), (3, 4), (5,)], rng.normal(size=600), ell=0.2, tuning=tun)


@pytest.mark.parametrize("items", ["auto", "single_cell"])
def test_all_points_in_one_cell(cuda, items):
    """One heavy cell: exercises work-item chunking (several chunks per supercell)."""
    tun = {"cell_items2": 1, "cell_items3": 1} if items == "single_cell" else None
    rng = np.random.default_rng(2)
    X = 0.001 + 1e-5 * rng.random(size=(5000, 3))
    _oracle_check(X, [(0, 1, 2), (0, 1), (2,)], rng.normal(size=5000), tuning=tun)


def test_clustered_data_many_chunks(cuda):
    rng = np.random.default_rng(3)
    X = np.concatenate([0.02 * rng.normal(size=(20000, 3)), rng.uniform(-0.14, 0.14, size=(3000, 3))])
    X = np.clip(X, -0.49, 0.49)
    _oracle_check(X, [(0, 1, 2)], rng.normal(size=X.shape[0]), ell=0.5)


def test_dense_2d_windows_tensor_core_items(cuda):
    """300k nodes in 2-D windows (mean occupancy ~70 per cell: single-cell tensor-core items
    chosen automatically) against the oracle and against the lane-per-point kernels."""
    rng = np.random.default_rng(7)
    X = rng.uniform(-0.5, 0.5, size=(300_000, 4))
    v = rng.normal(size=300_000)
    auto, _ = _oracle_check(X, [(0, 1), (2, 3), (1, 2)], v, family="matern12", ell=0.3)
    lane, _ = _oracle_check(X, [(0, 1), (2, 3), (1, 2)], v, family="matern12", ell=0.3, tuning={"cell_items2": 8})
    assert rel(auto, lane) <= 1e-13


@pytest.mark.parametrize("R", [2, 4, 6])
def test_rhs_pair_tensor_core_spread(cuda, R):
    """Even RHS counts on densely occupied 3-D windows take the RHS-pair tensor-core
    spread (k_spread3r): each column equals the one-RHS product (DFMA tile), the
    rhs_pair_spread=0 batch, and the oracle; footprints on the periodic boundary included."""
    from oracle import restate as R_
    from paper_2404_17344_b200.fastsum import build_plan, fast_matvec, fast_matvecs
    from paper_2404_17344_b200.kernels import KernelSpec
    from paper_2404_17344_b200.windows import WindowSet

    rng = np.random.default_rng(20 + R)
    N = 30_000
    X = np.concatenate([rng.uniform(-0.012, 0.012, size=(N // 2, 6)),
                        rng.uniform(-0.5, -0.49, size=(N - N // 2, 6))])   # centre and wrapping cells
    V = rng.normal(size=(R, N))
    ws = WindowSet(((1, 2, 3), (4, 5, 6)), d_max=3)
    plan = build_plan(KernelSpec("gauss", 0.3), ws, "default", _ds(X, 3))
    res = fast_matvecs(plan, V, dell=True)
    for r in range(R):
        assert rel(res["K"][r], fast_matvec(plan, V[r])) <= 1e-13
    ref = fast_matvecs(build_plan(KernelSpec("gauss", 0.3), ws, "default", _ds(X, 3), tuning={"rhs_pair_spread": 0}),
                       V, dell=True)
    assert rel(res["K"], ref["K"]) <= 1e-13 and rel(res["dK_dell"], ref["dK_dell"]) <= 1e-13
    orc = R_.FastSum("gauss", 0.3, 1.0, [(0, 1, 2), (3, 4, 5)], X).matvec(V[R - 1])
    assert rel(res["K"][R - 1], orc) <= 1e-8


@pytest.mark.parametrize("kernels", ["tuned", "generic"])
def test_row_masked_windows(cuda, kernels):
    """build_plan(row_masks=...) (ak_geom_create_masked): each window uses only its
    rows -- equal to plans built on the row subsets, zeros elsewhere; all-true masks
    equal the unmasked plan."""
    from dataclasses import replace

    from paper_2404_17344_b200.fastsum import build_plan, fast_matvecs
    from paper_2404_17344_b200.kernels import KernelSpec
    from paper_2404_17344_b200.windows import WindowSet

    tun = {"generic_kernels": 1} if kernels == "generic" else None
    rng = np.random.default_rng(31)
    N = 40_000
    X = rng.uniform(-0.14, 0.14, size=(N, 7))
    V = rng.normal(size=(2, N))
    ds = _ds(X, 3)
    ws = WindowSet(((1, 2, 3), (4, 5), (6,), (2, 4, 7)), d_max=3)
    spec = KernelSpec("gauss", 0.4)
    full = fast_matvecs(build_plan(spec, ws, "default", ds, tuning=tun), V, dell=True)
    ones = fast_matvecs(build_plan(spec, ws, "default", ds, row_masks=np.ones((4, N), bool), tuning=tun), V,
                        dell=True)
    assert rel(ones["K"], full["K"]) <= 1e-13 and rel(ones["dK_dell"], full["dK_dell"]) <= 1e-13
    masks = rng.random((4, N)) < np.array([0.3, 0.5, 0.7, 0.0])[:, None]
    masks[3, :5] = True                          # a nearly empty window
    masks[2] = False                             # an empty one
    got = fast_matvecs(build_plan(spec, ws, "default", ds, row_masks=masks, tuning=tun), V, dell=True)
    want = {k: np.zeros_like(got[k]) for k in ("K", "dK_dell")}
    for w, win in enumerate(ws.windows):
        rows = np.flatnonzero(masks[w])
        if not len(rows):
            continue
        sub = replace(ds, features=X[rows], targets=ds.targets[rows])
        part = fast_matvecs(build_plan(spec, WindowSet((win,), d_max=3), "default", sub, tuning=tun), V[:, rows],
                            dell=True)
        for k in want:
            want[k][:, rows] += part[k]
    assert rel(got["K"], want["K"]) <= 1e-13 and rel(got["dK_dell"], want["dK_dell"]) <= 1e-13


@pytest.mark.parametrize("preset", ["rough", "fine", 48])
def test_other_grid_sizes(cuda, preset):
    rng = np.random.default_rng(4)
    X = rng.uniform(-0.25, 0.25, size=(700, 6)) / math.sqrt(3)
    _oracle_check(X, [(0, 1, 2), (3, 4, 5), (1, 4), (2,)], rng.normal(size=700), preset=preset, ell=0.4)


@pytest.mark.parametrize("fam", ["gauss", "der_gauss", "matern12", "der_matern12"])
def test_families_q123(cuda, fam):
    rng = np.random.default_rng(6)
    X = rng.uniform(-0.25, 0.25, size=(900, 6)) / math.sqrt(3)
    _oracle_check(X, [(0, 1, 2), (3, 4), (5,), (0, 5)], rng.normal(size=900), family=fam, ell=0.35, sf=0.7)


def test_domain_error_from_device_check(cuda):
    from paper_2404_17344_b200.errors import PointOutOfDomainError
    from paper_2404_17344_b200.fastsum import build_plan
    from paper_2404_17344_b200.kernels import KernelSpec
    from paper_2404_17344_b200.windows import WindowSet

    X = np.zeros((10, 3))
    X[3, 1] = 0.5
    with pytest.raises(PointOutOfDomainError):
        build_plan(KernelSpec("gauss", 0.5), WindowSet(((1, 2, 3),), d_max=3), "default", _ds(X, 3))


def test_wrong_vector_length(cuda):
    from paper_2404_17344_b200.fastsum import build_plan, fast_matvec
    from paper_2404_17344_b200.kernels import KernelSpec
    from paper_2404_17344_b200.windows import WindowSet

    plan = build_plan(KernelSpec("gauss", 0.5), WindowSet(((1, 2),), d_max=2), "rough", _ds(np.zeros((5, 2)), 2))
    with pytest.raises(ValueError):
        fast_matvec(plan, np.ones(4))
    with pytest.raises(ValueError):
        fast_matvec(plan, np.ones((2, 5)))


@pytest.mark.parametrize("q", [1, 2, 3])
def test_adjointness(cuda, q):
    """<type2(c), w> = <c, conj(type1(w))> (reference test_nufft.py:162-175)."""
    from paper_2404_17344_b200.nufft import NufftPlan, nufft_type1, nufft_type2, prepare_points

    for m in (8, 16, 32):
        plan = NufftPlan(dims=q, m=m)
        for seed in range(5):
            rng = np.random.default_rng(seed)
            pts = rng.uniform(-0.5, 0.4999, size=(7, q))
            w = rng.normal(size=7) + 1j * rng.normal(size=7)
            c = rng.normal(size=(m,) * q) + 1j * rng.normal(size=(m,) * q)
            geom = prepare_points(plan, pts)
            lhs = np.sum(nufft_type2(plan, geom, c) * np.conj(w))
            rhs = np.sum(c * np.conj(nufft_type1(plan, geom, w)))
            assert abs(lhs - rhs) / max(abs(lhs), abs(rhs), 1e-30) <= 1e-8


def test_known_answers(cuda):
    from paper_2404_17344_b200.nufft import NufftPlan, nufft_type1, nufft_type2

    plan = NufftPlan(dims=2, m=8)
    c = np.zeros((8, 8), dtype=complex)
    c[0, 0] = 1.0
    pts = np.random.default_rng(0).uniform(-0.5, 0.5, size=(20, 2))
    np.testing.assert_allclose(nufft_type2(plan, pts, c), np.ones(20), atol=1e-9)
    np.testing.assert_allclose(nufft_type1(plan, np.array([[0.0, 0.0]]), np.array([1.0])), np.ones((8, 8)),
                               atol=1e-9)
    out = nufft_type1(NufftPlan(dims=1, m=8), np.random.default_rng(0).uniform(-0.5, 0.5, size=(5, 1)),
                      np.zeros(5))
    np.testing.assert_array_equal(out, np.zeros(8, dtype=complex))


def test_split_apply_and_grid_view(cuda):
    """spread_only + FROM_GRIDS equals one apply; the grid view aliases the op's buffer
    (the point-sharded multi-GPU path all-reduces exactly this view)."""
    from paper_2404_17344_b200 import _native
    from paper_2404_17344_b200.fastsum import build_plan
    from paper_2404_17344_b200.kernels import KernelSpec
    from paper_2404_17344_b200.windows import WindowSet

    rng = np.random.default_rng(8)
    X = rng.uniform(-0.25, 0.25, size=(3000, 6)) / math.sqrt(3)
    ws = WindowSet(((1, 2, 3), (4, 5), (6,)), d_max=3)
    plan = build_plan(KernelSpec("gauss", 0.4), ws, "default", _ds(X, 3))
    V = cuda.as_tensor(rng.normal(size=(2, 3000)), device="cuda")
    op = plan._operator(("gauss",), 2)
    ref = cuda.empty((2, 3000), dtype=cuda.float64, device="cuda")
    op.apply(V, [ref], [True])
    op.spread_only(V)
    g = op.grids()
    assert g.numel() == plan.geometries.canon_total * 2 and float(g.abs().sum()) > 0
    out = cuda.empty_like(ref)
    op.apply(None, [out], [True], flags=_native.AK_APPLY_FROM_GRIDS)
    assert rel(out.cpu().numpy(), ref.cpu().numpy()) <= 1e-15
    g.mul_(2.0)
    op.apply(None, [out], [True], flags=_native.AK_APPLY_FROM_GRIDS)
    assert rel(out.cpu().numpy(), 2.0 * ref.cpu().numpy()) <= 1e-15
    # band-spectrum exchange path (8x smaller all-reduce buffer)
    op.spectrum_only(V)
    b = op.band()
    m = plan.m
    assert b.numel() == 2 * 2 * (m * m * (m // 2) + m * (m // 2) + m // 2)
    op.apply(None, [out], [True], flags=_native.AK_APPLY_FROM_SPECTRUM)
    assert rel(out.cpu().numpy(), ref.cpu().numpy()) <= 1e-15
    b.mul_(3.0)
    op.apply(None, [out], [True], flags=_native.AK_APPLY_FROM_SPECTRUM)
    assert rel(out.cpu().numpy(), 3.0 * ref.cpu().numpy()) <= 1e-14


def test_sharded_plans_single_rank(cuda):
    """World size 1 (NCCL): both multi-GPU plans reproduce the single-GPU product."""
    import os
    import socket

    import torch.distributed as dist

    from paper_2404_17344_b200.distributed import PointShardedPlan, WindowShardedPlan
    from paper_2404_17344_b200.fastsum import build_plan, fast_matvec
    from paper_2404_17344_b200.kernels import KernelSpec
    from paper_2404_17344_b200.windows import WindowSet

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        rng = np.random.default_rng(10)
        X = rng.uniform(-0.25, 0.25, size=(5000, 7)) / math.sqrt(3)
        ws = WindowSet(((1, 2, 3), (4, 5, 6), (6, 7), (2,)), d_max=3)
        spec = KernelSpec("gauss", 0.5)
        ds = _ds(X, 3)
        v = rng.normal(size=5000)
        ref = fast_matvec(build_plan(spec, ws, "default", ds), v)
        vd = cuda.as_tensor(v, device="cuda")
        for make in (lambda: WindowShardedPlan(spec, ws, "default", ds),
                     lambda: PointShardedPlan(spec, ws, "default", ds),
                     lambda: PointShardedPlan(spec, ws, "default", ds, exchange="grid")):
            p = make()
            out = p.matvec(vd)
            assert rel(out.cpu().numpy(), ref) <= 1e-13, type(p).__name__
    finally:
        dist.destroy_process_group()


def test_side_stream_and_operator_cache(cuda):
    """Plan build and products on a non-default (non-blocking) stream match the default
    stream; the per-plan operator cache stays bounded."""
    import torch

    from paper_2404_17344_b200.fastsum import OPERATOR_CACHE_LIMIT, build_plan, fast_matvec, fast_matvecs
    from paper_2404_17344_b200.kernels import KernelSpec
    from paper_2404_17344_b200.windows import WindowSet

    rng = np.random.default_rng(8)
    X = rng.uniform(-0.14, 0.14, size=(3000, 5))
    v = rng.normal(size=3000)
    ws = WindowSet(((1, 2, 3), (4, 5), (2,)), d_max=3)
    spec = KernelSpec("gauss", 0.3)
    ref = fast_matvec(build_plan(spec, ws, "default", _ds(X, 3)), v)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        plan = build_plan(spec, ws, "default", _ds(X, 3))
        out = fast_matvec(plan, v)
        for R in range(1, OPERATOR_CACHE_LIMIT + 4):
            res = fast_matvecs(plan, np.tile(v, (R, 1)))
            assert rel(res["K"][-1], ref) <= 1e-13
    s.synchronize()
    assert rel(out, ref) <= 1e-13
    assert sum(1 for k in plan._cache if isinstance(k, tuple) and k[0] == "op") <= OPERATOR_CACHE_LIMIT


def test_q2_many_rhs(cuda):
    """2-D single-cell kernels with R = 11 right-hand sides: K V and dK/dl V rows equal
    the oracle's single products."""
    from oracle import restate as R
    from paper_2404_17344_b200.fastsum import build_plan, fast_matvecs
    from paper_2404_17344_b200.kernels import KernelSpec
    from paper_2404_17344_b200.windows import WindowSet

    rng = np.random.default_rng(9)
    X = rng.uniform(-0.1, 0.1, size=(20000, 4))
    V = rng.normal(size=(11, 20000))
    plan = build_plan(KernelSpec("matern12", 0.3), WindowSet(((1, 2), (3, 4)), d_max=2), "default", _ds(X, 2))
    res = fast_matvecs(plan, V, dell=True)
    for fam, key in (("matern12", "K"), ("der_matern12", "dK_dell")):
        fs = R.FastSum(fam, 0.3, 1.0, [(0, 1), (2, 3)], X)
        for r in (0, 7, 10):
            assert rel(res[key][r], fs.matvec(V[r])) <= 1e-8, (key, r)


def test_concurrent_streams_share_a_plan(cuda):
    """Two host threads, each on its own CUDA stream, run products on one plan at the
    same time: each stream gets its own operator workspace (results stay exact)."""
    import threading

    import torch

    from paper_2404_17344_b200.fastsum import build_plan, fast_matvec
    from paper_2404_17344_b200.kernels import KernelSpec
    from paper_2404_17344_b200.windows import WindowSet

    rng = np.random.default_rng(12)
    X = rng.uniform(-0.14, 0.14, size=(20000, 6))
    plan = build_plan(KernelSpec("gauss", 0.3), WindowSet(((1, 2, 3), (4, 5, 6)), d_max=3), "default", _ds(X, 3))
    vs = [torch.as_tensor(rng.normal(size=20000), device="cuda") for _ in range(2)]
    refs = [fast_matvec(plan, v).clone() for v in vs]
    torch.cuda.synchronize()
    outs, errors = [None, None], []

    def run(k):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for _ in range(20):
                    outs[k] = fast_matvec(plan, vs[k])
            s.synchronize()
        except Exception as exc:  # pragma: no cover - reported below
            errors.append(exc)

    threads = [threading.Thread(target=run, args=(k,)) for k in range(2)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for k in range(2):
        assert rel(outs[k].cpu().numpy(), refs[k].cpu().numpy()) <= 1e-13


def test_c5_full_size_properties(cuda):
    """Config 5 at its full size (4M nodes, 16 RHS, mixed windows and kernels):
    linearity across RHS, the per-window derivative outputs against single-window
    plans, operator symmetry, and dK/dsigma_f = 2/sigma_f K."""
    import torch

    from paper_2404_17344_b200 import configs
    from paper_2404_17344_b200.fastsum import build_mixed_plan, build_plan, fast_matvecs, mixed_matvecs
    from paper_2404_17344_b200.windows import WindowSet

    wl = configs.config5()
    plan = build_mixed_plan(wl.specs, wl.window_set, "default", wl.data)
    V = torch.as_tensor(wl.V, device="cuda")
    res = mixed_matvecs(plan, V)
    K = res["K"]
    # linearity: K(V0 - 2 V1) = K V0 - 2 K V1
    lin = mixed_matvecs(plan, (V[0] - 2.0 * V[1]).reshape(1, -1), dell=False, dsigma=False)["K"][0]
    scale = float(torch.max(torch.abs(K[0])))
    assert float(torch.max(torch.abs(lin - (K[0] - 2.0 * K[1])))) <= 1e-10 * scale
    # symmetry <K v0, v1> = <v0, K v1>
    lhs = float(torch.dot(K[0], V[1]))
    rhs_ = float(torch.dot(V[0], K[1]))
    assert abs(lhs - rhs_) <= 1e-8 * float(torch.linalg.vector_norm(V[0]) * torch.linalg.vector_norm(V[1]))
    assert rel(res["dK_dsigma"].cpu().numpy(), (2.0 / wl.specs[0].sigma_f) * K.cpu().numpy()) <= 1e-14
    # window 7 (2-D, Matern) and window 9 (1-D): per-window dK/dl against a single-window base plan
    for w in (6, 8):
        one = build_plan(wl.specs[w], WindowSet((wl.window_set.windows[w],), d_max=3), "default", wl.data)
        single = fast_matvecs(one, V[:2], dell=True)["dK_dell"]
        assert rel(res["dK_dell"][w][:2].cpu().numpy(), single.cpu().numpy()) <= 1e-12, w


def test_plans_release_device_memory(cuda):
    """Building and dropping plans (geometry, weight tables, operators, cuFFT plans) in a
    loop does not accumulate device memory."""
    import gc

    import torch

    from paper_2404_17344_b200.fastsum import build_plan, fast_matvecs
    from paper_2404_17344_b200.kernels import KernelSpec
    from paper_2404_17344_b200.windows import WindowSet

    rng = np.random.default_rng(17)
    X = rng.uniform(-0.05, 0.05, size=(50000, 6))
    V = rng.normal(size=(3, 50000))
    ws = WindowSet(((1, 2, 3), (4, 5), (6,)), d_max=3)

    def cycle():
        plan = build_plan(KernelSpec("gauss", 0.3), ws, "default", _ds(X, 3))
        fast_matvecs(plan, V, dell=True)
        del plan
        gc.collect()
        torch.cuda.synchronize()

    cycle()
    torch.cuda.empty_cache()
    free0 = torch.cuda.mem_get_info()[0]
    for _ in range(10):
        cycle()
    torch.cuda.empty_cache()
    free1 = torch.cuda.mem_get_info()[0]
    assert free0 - free1 < 64 * 2**20, (free0 - free1) / 2**20


@pytest.mark.parametrize("R", [8, 11, 16, 33])
def test_q1_rhs_lane_kernels(cuda, R):
    """R >= 8 RHS on 1-D windows run with the RHS across the lanes (k_spread1r /
    k_interp1r, RHS-minor data): every column equals the one-RHS product (lane-per-point
    kernels) and the oracle; per-window outputs (mixed plans) and the wrap-around
    boundary included; R = 33 spans two RHS chunks."""
    from oracle import restate as R_
    from paper_2404_17344_b200 import _native
    from paper_2404_17344_b200.fastsum import build_mixed_plan, build_plan, fast_matvec, fast_matvecs, mixed_matvecs
    from paper_2404_17344_b200.kernels import KernelSpec
    from paper_2404_17344_b200.windows import WindowSet

    rng = np.random.default_rng(40 + R)
    N = 60_000
    X = np.concatenate([rng.normal(scale=0.05, size=(N - 3000, 3)), rng.uniform(-0.5, -0.48, size=(3000, 3))])
    X = np.clip(X, -0.5, 0.49)
    V = rng.normal(size=(R, N))
    ws = WindowSet(((1,), (2,), (3,)), d_max=3)
    plan = build_plan(KernelSpec("matern12", 0.2), ws, "default", _ds(X, 3))
    with _native.KernelTimer() as kt:
        res = fast_matvecs(plan, V, dell=True)
    assert "k_spread1r" in kt.report and "k_interp1r" in kt.report, kt.report
    for r in (0, R // 2, R - 1):
        assert rel(res["K"][r], fast_matvec(plan, V[r])) <= 1e-13
    orc = R_.FastSum("matern12", 0.2, 1.0, [(0,), (1,), (2,)], X).matvec(V[R - 1])
    assert rel(res["K"][R - 1], orc) <= 1e-8
    mplan = build_mixed_plan([KernelSpec("matern12", 0.2), KernelSpec("gauss", 0.3), KernelSpec("matern12", 0.5)],
                             ws, "default", _ds(X, 3))
    mix = mixed_matvecs(mplan, V)
    for w, (fam, ell) in enumerate((("matern12", 0.2), ("gauss", 0.3), ("matern12", 0.5))):
        one = build_plan(KernelSpec(fam, ell), WindowSet((ws.windows[w],), d_max=3), "default", _ds(X, 3))
        col = fast_matvecs(one, V[R - 1], dell=True)["dK_dell"]
        assert rel(mix["dK_dell"][w][R - 1], col) <= 1e-13


@pytest.mark.parametrize("R", [8, 12, 16, 40])
def test_q2_rhs_batched_kernels(cuda, R):
    """R >= 8 RHS on densely occupied 2-D windows run one CTA per cell item for 8 RHS per
    warp (k_spread2r / k_interp2r, RHS-minor data): every column equals the one-RHS
    product (k_spread2c / k_interp2c) and the oracle; per-window outputs and wrapping
    footprints included; R = 12 and 40 leave partial warps / CTAs."""
    from oracle import restate as R_
    from paper_2404_17344_b200 import _native
    from paper_2404_17344_b200.fastsum import build_mixed_plan, build_plan, fast_matvec, fast_matvecs, mixed_matvecs
    from paper_2404_17344_b200.kernels import KernelSpec
    from paper_2404_17344_b200.windows import WindowSet

    rng = np.random.default_rng(60 + R)
    N = 50_000
    X = np.concatenate([rng.uniform(-0.1, 0.1, size=(N - 4000, 4)), rng.uniform(0.47, 0.5, size=(4000, 4))])
    X = np.minimum(X, np.nextafter(0.5, 0.0))
    V = rng.normal(size=(R, N))
    ws = WindowSet(((1, 2), (3, 4)), d_max=2)
    plan = build_plan(KernelSpec("gauss", 0.25), ws, "default", _ds(X, 2))
    with _native.KernelTimer() as kt:
        res = fast_matvecs(plan, V, dell=True)
    assert "k_spread2r" in kt.report and "k_interp2r" in kt.report, kt.report
    for r in (0, R // 2, R - 1):
        assert rel(res["K"][r], fast_matvec(plan, V[r])) <= 1e-13
    orc = R_.FastSum("gauss", 0.25, 1.0, [(0, 1), (2, 3)], X).matvec(V[R - 1])
    assert rel(res["K"][R - 1], orc) <= 1e-8
    dorc = R_.FastSum("der_gauss", 0.25, 1.0, [(0, 1), (2, 3)], X).matvec(V[0])
    assert rel(res["dK_dell"][0], dorc) <= 1e-8
    mplan = build_mixed_plan([KernelSpec("matern12", 0.2), KernelSpec("gauss", 0.3)], ws, "default", _ds(X, 2))
    mix = mixed_matvecs(mplan, V)
    for w, (fam, ell) in enumerate((("matern12", 0.2), ("gauss", 0.3))):
        one = build_plan(KernelSpec(fam, ell), WindowSet((ws.windows[w],), d_max=2), "default", _ds(X, 2))
        col = fast_matvecs(one, V[R - 1], dell=True)["dK_dell"]
        assert rel(mix["dK_dell"][w][R - 1], col) <= 1e-13
