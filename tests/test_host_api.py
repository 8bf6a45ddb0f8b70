"""Host-side API behaviour (no GPU): types, validation, plan-time tables,
the scaling pipeline and the window polynomial used by the CUDA kernels."""

import json
import math

import numpy as np
import pytest

from conftest import golden
from oracle import restate as R
from paper_2404_17344_b200 import dataset as D
from paper_2404_17344_b200 import kernels as K
from paper_2404_17344_b200 import nufft as NU
from paper_2404_17344_b200 import windows as W
from paper_2404_17344_b200.errors import (InvalidDMaxError, InvalidScalingError, PointOutOfDomainError)
from paper_2404_17344_b200 import fastsum as FS


def test_windowset_validation_and_json():
    ws = W.WindowSet(((1, 2, 3), (2, 5), (4,)), d_max=3, metadata={"technique": "x"})
    assert ws.lengths == (3, 2, 1)
    assert ws.columns((2, 5)) == [1, 4]
    assert ws.max_feature() == 5
    back = W.WindowSet.from_json(ws.to_json())
    assert back == ws and back.metadata == {"technique": "x"}
    assert json.loads(ws.to_json())["d_max"] == 3
    for bad in [((1, 1),), ((2, 1),), ((0, 1),), ((1, 2, 3, 4),), ()]:
        with pytest.raises(ValueError):
            W.WindowSet(bad, d_max=3)
    with pytest.raises(ValueError):
        W.WindowSet(((1,),), d_max=4)


def test_consec_and_singleton_windows():
    ws = W.consec_windows(8, 3)
    assert ws.windows == ((1, 2, 3), (4, 5, 6), (7, 8))
    assert W.singleton_windows(3).windows == ((1,), (2,), (3,))


def test_scaling_pipeline_matches_reference():
    g = golden("pipeline")
    ds = D.from_arrays(g["X"], g["y"])
    q = D.minmax_to_quarter_box(D.zscore_normalize(ds))
    p, ell = D.prescale(q, 2, 0.7)
    np.testing.assert_array_equal(p.features, g["prescaled"])
    np.testing.assert_array_equal(p.targets, g["targets"])
    assert ell == float(g["ell"])
    assert p.scaling_state == D.PRESCALED and p.d_max == 2
    with pytest.raises(InvalidScalingError):
        D.prescale(ds, 2, 1.0)
    with pytest.raises(InvalidDMaxError):
        D.prescale(q, 4, 1.0)
    with pytest.raises(InvalidScalingError):
        D.zscore_normalize(q)


def test_same_scaling_and_split():
    ds = D.from_arrays(np.random.default_rng(0).normal(size=(50, 3)), np.zeros(50))
    q = D.minmax_to_quarter_box(D.zscore_normalize(ds))
    p, _ = D.prescale(q, 2, 1.0)
    a, b = D.train_test_split(p, 0.6, seed=1)
    assert a.n_rows == 30 and b.n_rows == 20
    assert D.same_scaling(a, b)
    other = D.from_arrays(np.random.default_rng(1).normal(size=(50, 3)), np.zeros(50))
    p2, _ = D.prescale(D.minmax_to_quarter_box(D.zscore_normalize(other)), 2, 1.0)
    assert not D.same_scaling(p, p2)


def test_kernelspec_and_profiles():
    with pytest.raises(ValueError):
        K.KernelSpec("laplace", 1.0)
    with pytest.raises(ValueError):
        K.KernelSpec("gauss", 0.0)
    s = K.KernelSpec("gauss", 0.5, 2.0)
    assert s.operator_scale() == 4.0
    assert K.KernelSpec("der_gauss", 0.5, 2.0).operator_scale() == 4.0 * 2.0 / 0.5
    assert K.KernelSpec("der_matern12", 0.5, 1.0).operator_scale() == 2.0
    assert s.derivative().family == "der_gauss"
    assert K.eval_kernel(K.KernelSpec("der_gauss", 0.7), 2 * 0.7 * 0.7) == pytest.approx(math.exp(-1), abs=1e-15)
    r2 = np.linspace(0, 1, 17)
    for fam in K.FAMILIES:
        np.testing.assert_array_equal(K.radial_profile(fam, 0.3, r2), R.radial_profile(fam, 0.3, r2))


def test_resolve_m_and_presets():
    assert [FS.resolve_m(p) for p in ("fine", "default", "rough")] == [64, 32, 16]
    assert FS.resolve_m(24) == 24
    for bad in ("coarse", 15, 0):
        with pytest.raises(ValueError):
            FS.resolve_m(bad)


@pytest.mark.parametrize("q", [1, 2, 3])
@pytest.mark.parametrize("fam", K.FAMILIES)
def test_kernel_coefficients_match_oracle(q, fam):
    a = FS.kernel_coefficients(fam, 0.35, q, 16).values
    b = R.kernel_coefficients(fam, 0.35, q, 16)
    assert np.max(np.abs(a - b)) <= 1e-16 * max(1.0, np.max(np.abs(b))) * 10


def test_large_ell_constant_coefficient_dominates():
    t = FS.kernel_coefficients("gauss", 3.0, 1, 32).values
    assert abs(t[0]) > 100 * np.max(np.abs(t[1:]))


@pytest.mark.parametrize("m", [8, 16, 32, 64])
@pytest.mark.parametrize("window", ["kaiser_bessel", "gaussian_window"])
def test_nufft_plan_constants_match_oracle(m, window):
    p = NU.NufftPlan(3, m, window=window)
    o = R.Nufft(3, m, window=window)
    assert (p.n, p.beta) == (o.n, o.beta)
    np.testing.assert_allclose(p.deconvolution(), o.deconvolution(), rtol=1e-14)


@pytest.mark.parametrize("cutoff", [2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("window", ["kaiser_bessel", "gaussian_window"])
def test_window_polynomial_accuracy(cutoff, window):
    """The per-tap polynomial the kernels evaluate reproduces the window (abs, peak 1)."""
    p = NU.NufftPlan(2, 16, cutoff=cutoff, window=window)
    wf = p.window_fn()
    o = R.Nufft(2, 16, cutoff=cutoff, window=window)
    T = 2 * cutoff
    Tk = wf.taps                 # kernel taps: T, or T + 2 (zero outer taps, see PADDED_TAPS)
    k = (Tk - T) // 2
    assert Tk == NU.PADDED_TAPS.get(T, T)
    frac = np.linspace(0.0, 1.0, 1001, endpoint=False)
    s = 2 * frac - 1
    for a in range(Tk):
        pair = a if a < Tk // 2 else Tk - 1 - a
        e = np.polyval(np.array(wf.ce[pair][:]), s * s)
        od = np.polyval(np.array(wf.co[pair][:]), s * s)
        val = e + s * od if a < Tk // 2 else e - s * od
        if not k <= a < T + k:
            assert np.all(val == 0.0)  # padding tap: the reference has no tap there
            continue
        exact = o.window_values(frac + cutoff - 1 - (a - k))
        # ~1e-14 of the peak at the default cutoff 6; the 4-tap window is the roughest
        assert np.max(np.abs(val - exact)) < (NU.WINDOW_FIT_TOL_SMALL_CUTOFF if cutoff < 4 else 3e-14)


def test_band_multiplier_layout():
    p = NU.NufftPlan(3, 16)
    t = FS.kernel_coefficients("gauss", 0.3, 3, 16)
    H = FS.band_multiplier(t, p)
    assert H.shape == (16, 16, 8)
    d2 = 1.0 / p.window_transform(NU.freqs(16)) ** 2
    k = (3, 14, 5)
    assert H[k] == pytest.approx(t.values[k].real * d2[3] * d2[14] * d2[5], rel=1e-15)
    # H is even: H[k0,k1,k2] == H[-k0,-k1,k2] (with the zeroed -m/2 plane)
    assert H[1, 2, 3] == pytest.approx(H[15, 14, 3], rel=1e-12)
    assert np.all(H[8, :, :] == 0) and np.all(H[:, 8, :] == 0)


def test_nufft_plan_validation():
    with pytest.raises(ValueError):
        NU.NufftPlan(4, 8)
    with pytest.raises(ValueError):
        NU.NufftPlan(1, 7)
    with pytest.raises(ValueError):
        NU.NufftPlan(1, 8, cutoff=1)
    with pytest.raises(ValueError):
        NU.NufftPlan(1, 8, cutoff=9)  # > 16 taps: no GPU kernel
    with pytest.raises(ValueError):
        NU.CoefficientTable(dims=1, m=8, values=np.zeros(7))


def test_prepare_points_domain_check_is_host_side():
    p = NU.NufftPlan(1, 8)
    with pytest.raises(PointOutOfDomainError):
        NU.prepare_points(p, np.array([[0.5]]))
    with pytest.raises(PointOutOfDomainError):
        NU.prepare_points(p, np.array([[-0.6]]))


def test_build_plan_state_checks_before_device():
    rng = np.random.default_rng(0)
    ds = D.from_arrays(rng.normal(size=(40, 4)), np.zeros(40))
    q = D.minmax_to_quarter_box(D.zscore_normalize(ds))
    ws = W.WindowSet(((1, 2), (3, 4)), d_max=2)
    with pytest.raises(InvalidScalingError):
        FS.build_plan(K.KernelSpec("gauss", 0.5), ws, "default", q)
    p1, _ = D.prescale(q, 1, 1.0)
    with pytest.raises(InvalidScalingError):
        FS.build_plan(K.KernelSpec("gauss", 0.5), ws, "default", p1)


def test_eta_warning_emitted_before_device():
    ds = D.Dataset(np.zeros((3, 2)), np.zeros(3), ("a", "b"), scaling_state=D.PRESCALED, d_max=1)
    ws = W.WindowSet(((1,), (2,)), d_max=1)
    with pytest.warns(FS.AccuracyWarning):
        try:
            FS.build_plan(K.KernelSpec("gauss", 0.005), ws, "rough", ds)
        except Exception:
            pass  # no CUDA device here: the warning precedes the device work


def test_configs_shapes():
    from paper_2404_17344_b200 import configs

    w = configs.config1(100)
    assert w.data.features.shape == (100, 9) and w.V.shape == (1, 100)
    assert np.all(np.abs(w.data.features) <= 0.25 / math.sqrt(3) + 1e-15)
    w5 = configs.config5(200, rhs=2)
    assert w5.window_set.lengths == configs.C5_LENGTHS and w5.mixed
    assert [s.family for s in w5.specs] == ["gauss"] * 6 + ["matern12"] * 4


def test_empty_dataset_rejected_like_the_reference():
    """An empty training set never reaches the device: Dataset raises EmptyDatasetError
    (reference dataset.py, same check)."""
    from paper_2404_17344_b200.errors import EmptyDatasetError

    with pytest.raises(EmptyDatasetError):
        D.Dataset(np.zeros((0, 5)), np.zeros(0), tuple(f"x{i}" for i in range(5)), scaling_state=D.PRESCALED, d_max=3)


def test_plan_builders_reach_the_device_layer():
    """Every plan builder's host side runs up to the device allocation (a CPU-only
    host stops there): catches argument plumbing errors without a GPU."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("covered by the GPU tests")
    from paper_2404_17344_b200 import distributed as DI

    ds = D.Dataset(np.random.default_rng(0).uniform(-0.1, 0.1, size=(50, 3)), np.zeros(50), ("a", "b", "c"),
                   scaling_state=D.PRESCALED, d_max=2)
    ws = W.WindowSet(((1, 2), (3,)), d_max=2)
    spec = K.KernelSpec("gauss", 0.5)
    masks = np.ones((2, 50), dtype=bool)
    calls = [lambda: FS.build_plan(spec, ws, "default", ds),
             lambda: FS.build_plan(spec, ws, "default", ds, row_masks=masks),
             lambda: FS.build_mixed_plan([spec, K.KernelSpec("matern12", 0.3)], ws, "default", ds),
             lambda: FS.build_mixed_plan([spec, spec], ws, "default", ds, row_masks=masks)]
    for call in calls:
        with pytest.raises(Exception) as err:
            call()
        assert not isinstance(err.value, (NameError, TypeError, AttributeError)), err.value
    assert callable(DI.CellShardedPlan) and callable(DI.cell_partition)
