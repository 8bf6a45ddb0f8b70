"""Small cases that reach every kernel family of libaddkern_b200, each checked
against the oracle -- run against the checked library variant
(AK_LIB_PATH=paper_2404_17344_b200/libaddkern_b200_checked.so, tests/test_gpu_checked.py;
compute-sanitizer is closed on this GPU pool):

  * config-1 distribution, N=400, K + dK/dl (multi-cell q=3 items, fused transforms)
  * densely occupied cells, windows (3), (2), (1): single-cell q=3 spread / DMMA
    interp (TMA bulk copies + mbarriers), q=2 DMMA kernels, q=1 lane kernels
  * the same with 2 and 4 RHS (RHS-pair tensor-core spread k_spread3r)
  * a row-masked plan (ak_geom_create_masked)
  * sparse data with several RHS (supercell items, region tiles)
  * NUFFT type-1 / type-2 for q = 1..3 (cuFFT + extract / pad kernels)
  * dense GPU product (ak_dense_apply)
  * 16 RHS on a mixed-kernel plan (RHS-minor batched kernels, RHS-pair spread)
"""

from __future__ import annotations

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - b) / max(np.linalg.norm(b), 1e-300))


def main():
    import torch

    from oracle import restate as R
    from paper_2404_17344_b200 import configs, nufft
    from paper_2404_17344_b200.dataset import PRESCALED, Dataset
    from paper_2404_17344_b200.fastsum import build_plan, fast_matvecs
    from paper_2404_17344_b200.kernels import KernelSpec, dense_matvec
    from paper_2404_17344_b200.windows import WindowSet

    torch.cuda.set_device(0)
    worst = 0.0

    wl = configs.config1(400)
    plan = build_plan(wl.spec, wl.window_set, "default", wl.data)
    res = fast_matvecs(plan, wl.V, dell=True)
    cols = [wl.window_set.columns(w) for w in wl.window_set]
    ref = R.FastSum("gauss", wl.spec.ell, 1.0, cols, wl.data.features).matvec(wl.V[0])
    worst = max(worst, rel(res["K"][0], ref))
    print("config1 K", rel(res["K"][0], ref), flush=True)

    rng = np.random.default_rng(5)
    N = 2000
    X = rng.uniform(-0.01, 0.01, size=(N, 6))
    ds = Dataset(X, np.zeros(N), tuple(f"x{i}" for i in range(6)), scaling_state=PRESCALED, d_max=3)
    ws = WindowSet(((1, 2, 3), (4, 5), (6,)), d_max=3)
    dplan = build_plan(KernelSpec("gauss", 0.3), ws, "default", ds)
    for Rn in (1, 2, 4):
        V = rng.normal(size=(Rn, N))
        out = fast_matvecs(dplan, V, dell=True)
        for r in range(Rn):
            refr = R.FastSum("gauss", 0.3, 1.0, [(0, 1, 2), (3, 4), (5,)], X).matvec(V[r])
            e = rel(out["K"][r], refr)
            worst = max(worst, e)
        print(f"dense cells R={Rn} K", e, flush=True)

    masks = rng.random((3, N)) < 0.6
    mplan = build_plan(KernelSpec("gauss", 0.3), ws, "default", ds, row_masks=masks)
    v = rng.normal(size=N)
    out = fast_matvecs(mplan, v)["K"]
    ref = np.zeros(N)
    for k, w in enumerate([(0, 1, 2), (3, 4), (5,)]):
        rows = np.flatnonzero(masks[k])
        part = R.FastSum("gauss", 0.3, 1.0, [w], X[rows]).matvec(v[rows])
        ref[rows] += part
    worst = max(worst, rel(out, ref))
    print("masked K", rel(out, ref), flush=True)

    Xs = rng.uniform(-0.14, 0.14, size=(3000, 6))
    dss = Dataset(Xs, np.zeros(3000), tuple(f"x{i}" for i in range(6)), scaling_state=PRESCALED, d_max=3)
    splan = build_plan(KernelSpec("gauss", 0.5), WindowSet(((1, 2, 3), (4, 5, 6)), d_max=3), "default", dss)
    V = rng.normal(size=(3, 3000))
    out = fast_matvecs(splan, V, dell=True)["dK_dell"]
    refd = R.FastSum("der_gauss", 0.5, 1.0, [(0, 1, 2), (3, 4, 5)], Xs).matvec(V[2])
    worst = max(worst, rel(out[2], refd))
    print("sparse dK", rel(out[2], refd), flush=True)
    # sparse supercell items with 8 RHS per CTA (k_spread3b), two RHS chunks
    V16 = rng.normal(size=(16, 3000))
    out = fast_matvecs(splan, V16)["K"]
    for r in (0, 15):
        refr = R.FastSum("gauss", 0.5, 1.0, [(0, 1, 2), (3, 4, 5)], Xs).matvec(V16[r])
        worst = max(worst, rel(out[r], refr))
    print("sparse R=16 K", rel(out[15], refr), flush=True)

    # many RHS (RHS-minor batched kernels: k_spread1r / k_interp1r, k_spread2r / k_interp2r,
    # RHS-pair k_spread3r), mixed kernels with per-window outputs, boundary-hugging nodes
    from paper_2404_17344_b200.fastsum import build_mixed_plan, mixed_matvecs
    Xm = np.concatenate([rng.uniform(-0.02, 0.02, size=(5000, 6)), rng.uniform(-0.5, -0.48, size=(500, 6))])
    dsm = Dataset(Xm, np.zeros(len(Xm)), tuple(f"x{i}" for i in range(6)), scaling_state=PRESCALED, d_max=3)
    wsm = WindowSet(((1, 2, 3), (4, 5), (6,)), d_max=3)
    specs = [KernelSpec("gauss", 0.3), KernelSpec("matern12", 0.4), KernelSpec("matern12", 0.2)]
    Vm = rng.normal(size=(16, len(Xm)))
    res = mixed_matvecs(build_mixed_plan(specs, wsm, "default", dsm), Vm)
    refm = np.zeros(len(Xm))
    for (fam, ell), w in zip((("gauss", 0.3), ("matern12", 0.4), ("matern12", 0.2)), [(0, 1, 2), (3, 4), (5,)]):
        refm += R.FastSum(fam, ell, 1.0, [w], Xm).matvec(Vm[15])
    worst = max(worst, rel(res["K"][15], refm))
    print("mixed R=16 K", rel(res["K"][15], refm), flush=True)

    for q in (1, 2, 3):
        np_ = nufft.NufftPlan(dims=q, m=16)
        pts = rng.uniform(-0.5, 0.5, size=(300, q))
        w = rng.normal(size=300) + 1j * rng.normal(size=300)
        S = nufft.nufft_type1(np_, pts, w)
        op = R.Nufft(q, 16)
        Sref = R.type1(op, R.Geometry(op, pts), w)
        f = nufft.nufft_type2(np_, pts, Sref)
        fref = R.type2(op, R.Geometry(op, pts), Sref)
        worst = max(worst, rel(S, Sref), rel(f, fref))
        print(f"nufft q={q}", rel(S, Sref), rel(f, fref), flush=True)

    d = dense_matvec(KernelSpec("gauss", 0.5), WindowSet(((1, 2, 3), (4, 5, 6)), d_max=3), dss, V[0][:3000])
    dref = R.dense_matvec("gauss", 0.5, 1.0, [(0, 1, 2), (3, 4, 5)], Xs, V[0])
    worst = max(worst, rel(d, dref))
    print("dense", rel(d, dref), flush=True)
    torch.cuda.synchronize()
    print(f"SANITIZE_CASES_OK worst={worst:.3e}", flush=True)
    assert worst <= 1e-8


if __name__ == "__main__":
    main()
