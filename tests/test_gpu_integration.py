"""GPU: the INTEGRATION.md ctypes stub, verbatim, against the reference's golden
vectors.  The stub binds libaddkern_b200 through its C ABI only (numpy inputs,
torch for device buffers), the way an `addkern` maintainer would replace the
numba kernels behind `addkern.fastsum`."""

import numpy as np
import pytest

from conftest import golden, rel

pytestmark = pytest.mark.gpu

# --- INTEGRATION.md stub (keep in sync) -------------------------------------------
import ctypes  # noqa: E402


def b200_plan(features, windows, family, ell, sigma_f, m=32, cutoff=6):
    """replaces build_plan's geometry + tables (fastsum.py:105-133); windows 1-based."""
    import torch

    from paper_2404_17344_b200 import _native
    from paper_2404_17344_b200.fastsum import band_multiplier, kernel_coefficients
    from paper_2404_17344_b200.kernels import KernelSpec
    from paper_2404_17344_b200.nufft import NufftPlan

    lib = _native.lib()
    X = torch.as_tensor(np.ascontiguousarray(features, dtype=np.float64), device="cuda")
    P = len(windows)
    nplans = {len(w): NufftPlan(dims=len(w), m=m, cutoff=cutoff) for w in windows}
    n = next(iter(nplans.values())).n
    wf = next(iter(nplans.values())).window_fn()          # per-tap window polynomials
    q = (ctypes.c_int32 * P)(*[len(w) for w in windows])
    cols = []
    for w in windows:
        cols += [c - 1 for c in w] + [0] * (3 - len(w))
    geom = ctypes.c_void_p()
    _native.check(lib.ak_geom_create(n, P, q, (ctypes.c_int32 * (3 * P))(*cols), ctypes.c_void_p(X.data_ptr()),
                                     X.shape[0], X.shape[1], ctypes.byref(wf), None, ctypes.byref(geom)),
                  "ak_geom_create")
    op = ctypes.c_void_p()
    _native.check(lib.ak_op_create(geom, None, m, 1, 1, None, ctypes.byref(op)), "ak_op_create")
    H = {qq: torch.as_tensor(band_multiplier(kernel_coefficients(family, ell, qq, m), p).ravel(), device="cuda")
         for qq, p in nplans.items()}
    Hptr = torch.as_tensor(np.array([H[len(w)].data_ptr() for w in windows], dtype=np.int64), device="cuda")
    scale = torch.full((P,), KernelSpec(family, ell, sigma_f).operator_scale(), dtype=torch.float64, device="cuda")
    return {"geom": geom, "op": op, "H": H, "Hptr": Hptr, "scale": scale, "N": X.shape[0]}


def b200_fast_matvec(plan, v):
    """replaces fast_matvec's window loop (fastsum.py:150-160): numpy in, numpy out."""
    import torch

    from paper_2404_17344_b200 import _native

    N = plan["N"]
    V = torch.as_tensor(np.asarray(v, dtype=np.float64), device="cuda").reshape(1, N)
    out = torch.empty((1, N), dtype=torch.float64, device="cuda")
    _native.check(_native.lib().ak_op_apply(plan["op"], V.data_ptr(), N, plan["Hptr"].data_ptr(),
                                            plan["scale"].data_ptr(), (ctypes.c_void_p * 1)(out.data_ptr()), N,
                                            (ctypes.c_int32 * 1)(1), 0, None), "ak_op_apply")
    return out[0].cpu().numpy()


def b200_free(plan):
    from paper_2404_17344_b200 import _native

    _native.lib().ak_op_destroy(plan["op"])
    _native.lib().ak_geom_destroy(plan["geom"])
# --- end of stub --------------------------------------------------------------------


@pytest.mark.parametrize("name", ["c1", "c2", "c4"])
def test_integration_stub_matches_reference(cuda, name):
    g = golden(name)
    windows = [tuple(int(c) for c in row[:q]) for row, q in zip(g["windows"], g["lengths"])]
    plan = b200_plan(g["X"], windows, str(g["families"][0]), float(g["ells"][0]), float(g["sigma_f"]))
    try:
        for r, v in enumerate(g["V"]):
            assert rel(b200_fast_matvec(plan, v), g["K_default"][r]) <= 1e-8
    finally:
        b200_free(plan)
