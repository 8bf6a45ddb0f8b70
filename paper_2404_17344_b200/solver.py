"""CG kernel ridge regression on the GPU operator (the first caller of the hot path).

Mirrors ``addkern.solver`` (/root/reference/pkg/src/addkern/solver.py):
``cg_solve`` (:43-80, unpreconditioned CG on (A + beta I) v = y, relative
residual tolerance, CgBreakdownError / MaxIterationsError), ``krr_fit``
(:99-120), ``krr_predict`` (:123-132) and ``grid_search`` (:157-198).

Differences in where the work runs, not in what is computed:
* vectors stay on the device (torch) for the fast-summation backend; each CG
  iteration is one ``ak_op_apply`` plus a few vector ops and one host read of
  the residual norm (the reference's per-iteration stopping test);
* ``grid_search`` runs all (ell, beta) cells' CG iterations in lockstep as ONE
  batched operator over a single bin-sorted geometry: right-hand side r of the
  batch is cell r's search direction and uses cell r's band multiplier
  (``AK_APPLY_H_PER_RHS``).  The reference rebuilds the plan for every cell
  (solver.py:179-183) although the geometry does not depend on ell or beta.
  Converged or failed cells are frozen, so every cell performs exactly the
  iterations a standalone ``krr_fit`` would.
"""

from __future__ import annotations

import math
import time
import warnings
from dataclasses import dataclass, field

import numpy as np

from .dataset import PRESCALED, Dataset, same_scaling
from .errors import (CgBreakdownError, InvalidScalingError, MaxIterationsError, NativeLibraryError,
                     ScalingMismatchError)
from .kernels import KernelSpec, dense_cross_matvec, dense_matvec
from .windows import WindowSet

DEFAULT_CG_TOL = 1e-3
DEFAULT_CG_MAX_ITER = 5000
#: long krr_fit solves replay the CG iteration as a captured CUDA graph (eager launches of the
#: same iteration if the product cannot be captured)
GRAPHED_CG = True
#: CG iterations between host reads of the device-side CG state
CG_CHECK_EVERY = 8
#: iterations launched eagerly before the iteration is captured as a CUDA graph: the capture
#: costs ~6 ms and a replayed iteration saves ~0.02 ms over an eager one (B200, N = 20k .. 1M),
#: so only solves with some 300 iterations still to run gain from it
CG_GRAPH_AFTER = 256

DENSE = "dense"
FASTSUM = "fastsum"


def rmse(y_true, y_pred) -> float:
    a = np.asarray(y_true, dtype=np.float64).ravel()
    b = np.asarray(y_pred, dtype=np.float64).ravel()
    return float(np.sqrt(np.mean((a - b) ** 2)))


def default_sigma_f(n_windows: int) -> float:
    """sigma_f = sqrt(1/P) normalises the additive kernel's diagonal to 1 (solver.py:38-40)."""
    return math.sqrt(1.0 / n_windows)


def _is_tensor(x) -> bool:
    try:
        import torch

        return isinstance(x, torch.Tensor)
    except ImportError:  # pragma: no cover
        return False


def cg_solve(matvec, y, beta: float, tol: float = DEFAULT_CG_TOL, max_iter: int = DEFAULT_CG_MAX_ITER,
             callback=None):
    """Solve (A + beta I) v = y, A symmetric PSD; returns (v, iterations) (solver.py:43-80).

    ``y`` may be a numpy vector (matvec maps numpy -> numpy) or a torch CUDA
    tensor (matvec maps tensors -> tensors; every vector stays on the device).
    """
    if _is_tensor(y):
        return _cg_solve_device(matvec, y, beta, tol, max_iter, callback)
    else:
        y = np.asarray(y, dtype=np.float64)
        dot = lambda a, b: float(a @ b)
        norm = lambda a: float(np.linalg.norm(a))
        x = np.zeros_like(y)
        copy = np.copy
    y_norm = norm(y)
    if y_norm == 0.0:
        return x, 0
    r = copy(y)
    p = copy(r)
    rs = dot(r, r)
    if callback is not None:
        callback(math.sqrt(rs))
    if math.sqrt(rs) <= tol * y_norm:
        return x, 0
    for it in range(1, max_iter + 1):
        Ap = matvec(p) + beta * p
        pAp = dot(p, Ap)
        if pAp <= 0.0:
            raise CgBreakdownError(f"p^T A p = {pAp:.3e} <= 0 at iteration {it}")
        alpha = rs / pAp
        x += alpha * p
        r -= alpha * Ap
        rs_new = dot(r, r)
        if callback is not None:
            callback(math.sqrt(rs_new))
        if math.sqrt(rs_new) <= tol * y_norm:
            return x, it
        p = r + (rs_new / rs) * p
        rs = rs_new
    raise MaxIterationsError(f"CG did not reach tol={tol} within {max_iter} iterations")


def _cg_solve_graphed(matvec, y, beta, tol, max_iter, callback):
    """cg_solve on the device with one CG iteration = the product plus the native
    `ak_cg_step` (dots, vector updates, convergence / breakdown tests, iteration count and
    residual history, all on the device; solver.py:43-80 of the reference).

    The step does nothing once the residual test has passed or p^T A p <= 0, so the host
    reads the state only every CG_CHECK_EVERY iterations: the round trip that a
    per-iteration test costs (20-45% of an iteration below N = 100k) is paid once per
    CG_CHECK_EVERY iterations, and the result, the iteration count and the callback
    values are exactly those of the iteration-by-iteration loop (at most
    CG_CHECK_EVERY - 1 no-op iterations at the end).  The first CG_GRAPH_AFTER
    iterations are launched eagerly (capturing a graph costs ~6 ms, more than a short
    solve); a solve that is still running then captures the iteration as a CUDA graph
    and replays it (one launch per iteration instead of the product's ~0.13 ms of host
    launch work).  The callback is invoked with the whole residual history once the
    solve ends."""
    import torch

    from . import _native

    y = y.to(torch.float64).contiguous()
    x = torch.zeros_like(y)
    y_norm = float(torch.linalg.vector_norm(y))
    if y_norm == 0.0:
        return x, 0
    r = y.clone()
    p = r.clone()
    rs_h = float(torch.dot(r, r))
    if callback is not None:
        callback(math.sqrt(rs_h))
    if math.sqrt(rs_h) <= tol * y_norm:
        return x, 0
    n = y.numel()
    init = [0.0] * _native.AK_CG_STATE
    init[_native.AK_CG_RS] = rs_h
    init[_native.AK_CG_ACTIVE] = 1.0
    init[_native.AK_CG_THRESHOLD] = tol * y_norm
    state = torch.tensor(init, dtype=torch.float64, device=y.device)
    hist = torch.zeros(max_iter + 1, dtype=torch.float64, device=y.device)
    work = torch.empty(_native.AK_CG_WORK, dtype=torch.float64, device=y.device)
    lib = _native.lib()

    def step(Kp):
        Kp = Kp.contiguous()
        _native.check(lib.ak_cg_step(Kp.data_ptr(), float(beta), x.data_ptr(), r.data_ptr(), p.data_ptr(), n,
                                     state.data_ptr(), hist.data_ptr(), hist.numel(), work.data_ptr(),
                                     torch.cuda.current_stream().cuda_stream), "ak_cg_step")

    def capture():
        """The iteration as a CUDA graph (None if the product cannot be captured)."""
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        try:
            with torch.cuda.stream(s):
                matvec(p)                     # operators / cuFFT plans exist on this stream before capture
                torch.cuda.current_stream().synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    step(matvec(p))
        except RuntimeError as exc:
            # capture refused (e.g. an op the capture cannot record): stay with eager
            # launches of the same iteration.  Library, allocation and argument errors propagate.
            torch.cuda.current_stream().wait_stream(s)
            if isinstance(exc, NativeLibraryError) or "out of memory" in str(exc):
                raise
            warnings.warn(f"CUDA-graph capture of the CG iteration failed ({exc}); running it eagerly",
                          RuntimeWarning, stacklevel=4)
            return None
        torch.cuda.current_stream().wait_stream(s)
        return g

    def report(upto):
        if callback is not None and upto >= 1:
            for rs_it in hist[1:upto + 1].tolist():
                callback(math.sqrt(rs_it))

    done = 0
    graph, try_graph = None, GRAPHED_CG
    while done < max_iter:
        k = min(CG_CHECK_EVERY, max_iter - done)
        if try_graph and done >= CG_GRAPH_AFTER:
            graph, try_graph = capture(), False
        for _ in range(k):
            if graph is not None:
                graph.replay()
            else:
                step(matvec(p))
        done += k
        st = state.tolist()                   # one host read per CG_CHECK_EVERY iterations
        iters = int(st[_native.AK_CG_ITERATIONS])
        if st[_native.AK_CG_BREAKDOWN_AT] > 0.0:
            report(iters)
            raise CgBreakdownError(f"p^T A p = {st[_native.AK_CG_BREAKDOWN_PAP]:.3e} <= 0 "
                                   f"at iteration {int(st[_native.AK_CG_BREAKDOWN_AT])}")
        if st[_native.AK_CG_ACTIVE] == 0.0:
            report(iters)
            return x, iters
    report(max_iter)
    raise MaxIterationsError(f"CG did not reach tol={tol} within {max_iter} iterations")


def _cg_solve_device(matvec, y, beta, tol, max_iter, callback):
    """cg_solve on CUDA tensors with the scalars kept on the device: one host read per
    iteration (p^T A p and the new residual norm together) instead of two, and no
    host round trip between the vector updates.  Same arithmetic as the host loop:
    alpha = rs / pAp, x += alpha p, r -= alpha Ap, p = r + (rs_new / rs) p.  On a
    breakdown the (discarded) update of that iteration is computed before the
    check; the error is raised exactly where the reference raises it."""
    import torch

    y = y.to(torch.float64)
    x = torch.zeros_like(y)
    y_norm = float(torch.linalg.vector_norm(y))
    if y_norm == 0.0:
        return x, 0
    r = y.clone()
    p = r.clone()
    rs = torch.dot(r, r)
    rs_h = float(rs)
    if callback is not None:
        callback(math.sqrt(rs_h))
    if math.sqrt(rs_h) <= tol * y_norm:
        return x, 0
    for it in range(1, max_iter + 1):
        Ap = matvec(p) + beta * p
        pAp = torch.dot(p, Ap)
        alpha = rs / pAp
        x.add_(alpha * p)
        r.sub_(alpha * Ap)
        rs_new = torch.dot(r, r)
        pAp_h, rs_new_h = torch.stack([pAp, rs_new]).tolist()
        if pAp_h <= 0.0:
            raise CgBreakdownError(f"p^T A p = {pAp_h:.3e} <= 0 at iteration {it}")
        if callback is not None:
            callback(math.sqrt(rs_new_h))
        if math.sqrt(rs_new_h) <= tol * y_norm:
            return x, it
        p.mul_(rs_new / rs).add_(r)
        rs = rs_new
    raise MaxIterationsError(f"CG did not reach tol={tol} within {max_iter} iterations")


@dataclass(frozen=True)
class KrrModel:
    """Fitted ridge-regression state (solver.py:83-96)."""

    spec: KernelSpec
    window_set: WindowSet
    beta: float
    backend: str
    preset: object
    coefficients: np.ndarray
    train: Dataset
    cg_iterations: int
    residual: float
    plan: object = field(default=None, repr=False, compare=False)


def krr_fit(train: Dataset, ws: WindowSet, spec: KernelSpec, beta: float, backend: str = FASTSUM,
            preset="default", tol: float = DEFAULT_CG_TOL, max_iter: int = DEFAULT_CG_MAX_ITER) -> KrrModel:
    """Solve (K + beta I) v = y on the training set (solver.py:99-120)."""
    if train.scaling_state != PRESCALED:
        raise InvalidScalingError("krr_fit requires prescaled training data")
    log = []
    plan = None
    if backend == FASTSUM:
        import torch

        from .fastsum import build_plan, fast_matvec

        plan = build_plan(spec, ws, preset, train)
        y = torch.as_tensor(train.targets, device="cuda")
        v, iters = _cg_solve_graphed(lambda p: fast_matvec(plan, p), y, beta, tol, max_iter, log.append)
        coef = v.cpu().numpy()
    elif backend == DENSE:
        coef, iters = cg_solve(lambda p: dense_matvec(spec, ws, train, p), train.targets, beta, tol=tol,
                               max_iter=max_iter, callback=log.append)
    else:
        raise ValueError(f"unknown backend {backend!r}")
    y_norm = float(np.linalg.norm(train.targets))
    residual = log[-1] / y_norm if y_norm > 0 else 0.0
    return KrrModel(spec=spec, window_set=ws, beta=beta, backend=backend, preset=preset, coefficients=coef,
                    train=train, cg_iterations=iters, residual=float(residual), plan=plan)


def krr_predict(model: KrrModel, test: Dataset) -> np.ndarray:
    """h(x') = sum_j v_j kappa(x', x_j) through the fitted backend (solver.py:123-132)."""
    if test.scaling_state != PRESCALED or not same_scaling(model.train, test):
        raise ScalingMismatchError("test data must be prescaled with the training maps")
    if model.backend == DENSE:
        return dense_cross_matvec(model.spec, model.window_set, test, model.train, model.coefficients)
    from .fastsum import fast_cross_matvec, prepare_eval_points

    geoms = prepare_eval_points(model.plan, test)
    return fast_cross_matvec(model.plan, geoms, model.coefficients, test.n_rows)


@dataclass(frozen=True)
class GridCell:
    ell: float
    beta: float
    rmse: float | None
    cg_iterations: int | None
    fit_seconds: float
    predict_seconds: float
    failed: bool = False
    message: str = ""


@dataclass(frozen=True)
class GridSearchResult:
    cells: tuple
    best: GridCell

    @property
    def best_pair(self) -> tuple:
        return self.best.ell, self.best.beta


def _grid_operator(plan, specs, R, interp_geom=None):
    """One batched operator whose RHS r uses cell r's band multiplier."""
    from .fastsum import _Operator, band_multiplier, kernel_coefficients

    per_q = {}
    H = []
    for spec in specs:
        for w in plan.window_set:
            q = len(w)
            key = (spec.family, spec.ell, q)
            if key not in per_q:
                per_q[key] = band_multiplier(kernel_coefficients(spec.family, spec.ell, q, plan.m),
                                             plan.nufft_plans[q])
            H.append(per_q[key])
    scales = [specs[0].operator_scale()] * len(plan.window_set)
    gi = interp_geom if interp_geom is not None else plan.geometries
    return _Operator(plan.geometries, gi, plan.m, R, [H], [scales], per_rhs=True)


def _subset_applier(plan, specs, full_op):
    """apply_subset for cg_solve_batched over a per-RHS grid operator: products for the
    active cells only, on operators of power-of-two batch size (cached; padding rows
    are zero directions) whose per-RHS multiplier tables are re-pointed at the active
    cells' tables of `full_op` (which keeps them alive)."""
    import torch

    R, P = full_op.R, full_op.P
    table = full_op.hptr.reshape(R, P)
    ops = {R: full_op}

    def bucket(n):
        b = 1
        while b < n:
            b *= 2
        return min(b, R)

    def bind(idx):
        """The product for a fixed active set: operator bucket, multiplier tables and the
        padded input buffer prepared once."""
        n = len(idx)
        B = bucket(n)
        op = ops.get(B)
        if op is None:
            op = _grid_operator(plan, specs[:B], B)
            ops[B] = op
        rows = np.concatenate([idx, np.full(B - n, idx[0])]) if B > n else idx
        tables = table[torch.as_tensor(rows, device=table.device)].reshape(-1)
        Pp = [None]

        def product(Pa):
            op.set_rhs_multipliers(tables)   # buckets are shared between active sets
            if B > n:
                if Pp[0] is None:
                    Pp[0] = torch.zeros((B, Pa.shape[1]), dtype=Pa.dtype, device=Pa.device)
                Pp[0][:n] = Pa
                src = Pp[0]
            else:
                src = Pa
            out = torch.empty_like(src)
            op.apply(src, [out], [True])
            return out[:n]

        return product

    def apply_subset(Pa, idx):
        return bind(idx)(Pa)

    apply_subset.bind = bind
    return apply_subset


def cg_solve_batched(apply, Y, betas, tol: float = DEFAULT_CG_TOL, max_iter: int = DEFAULT_CG_MAX_ITER,
                     apply_subset=None):
    """Lockstep CG for R independent systems (A_r + beta_r I) x_r = y_r on the device.

    ``apply`` maps an (R, N) tensor of directions to (A_r p_r)_r.  If
    ``apply_subset(P_active, idx)`` is given, only the still-active systems are
    multiplied ((R_active, N) -> (R_active, N), idx = their indices), so
    converged systems stop costing products; an ``apply_subset.bind(idx)`` method,
    if present, returns the product for a fixed active set (per-set preparation
    done once).  Returns (X, iterations, messages); iterations[r] = -1 for a
    failed system, whose message says why.  Each system follows exactly the
    iteration of cg_solve.

    Everything after the product is the native `ak_cg_step_batched` (per-system
    dots, updates, convergence / breakdown tests and iteration counts on the
    device); the host reads the systems' states and compacts the active set every
    CG_CHECK_EVERY iterations -- systems that end in between are skipped by the
    step and merely ride along in the product until then.
    """
    import torch

    from . import _native

    R, N = Y.shape
    Y = Y.to(torch.float64).contiguous()
    dev = Y.device
    betas_d = torch.as_tensor(np.asarray(betas, dtype=np.float64), device=dev).reshape(R).contiguous()
    X = torch.zeros_like(Y)
    Rr = Y.clone()
    P = Rr.clone()
    yn = torch.linalg.vector_norm(Y, dim=1).cpu().numpy()
    rs_h = (Rr * Rr).sum(dim=1).cpu().numpy()
    iters = np.full(R, -1, dtype=np.int64)
    msgs = [""] * R
    active = np.ones(R, dtype=bool)
    for r in range(R):
        if yn[r] == 0.0 or math.sqrt(rs_h[r]) <= tol * yn[r]:
            iters[r] = 0
            active[r] = False
    init = np.zeros((R, _native.AK_CG_STATE))
    init[:, _native.AK_CG_RS] = rs_h
    init[:, _native.AK_CG_ACTIVE] = active
    init[:, _native.AK_CG_THRESHOLD] = tol * yn
    state = torch.as_tensor(init, device=dev)
    work = torch.empty(R * _native.AK_CG_WORK, dtype=torch.float64, device=dev)
    lib = _native.lib()
    done = 0
    while done < max_iter and active.any():
        idx = np.nonzero(active)[0]
        idx_d = torch.as_tensor(idx, device=dev)
        slots = torch.as_tensor(idx.astype(np.int32), device=dev)
        if apply_subset is None:
            product = None
        elif hasattr(apply_subset, "bind"):
            product = apply_subset.bind(idx)
        else:
            product = lambda Pa, idx=idx: apply_subset(Pa, idx)  # noqa: E731
        k = min(CG_CHECK_EVERY, max_iter - done)
        for _ in range(k):
            if product is None:
                Kp = apply(P).contiguous()
                slot_ptr, B = 0, R                      # slot r is system r
            else:
                Kp = product(P.index_select(0, idx_d)).contiguous()
                slot_ptr, B = slots.data_ptr(), len(idx)
            _native.check(lib.ak_cg_step_batched(Kp.data_ptr(), slot_ptr, B, betas_d.data_ptr(), X.data_ptr(),
                                                 Rr.data_ptr(), P.data_ptr(), N, state.data_ptr(), 0, 0,
                                                 work.data_ptr(), torch.cuda.current_stream().cuda_stream),
                          "ak_cg_step_batched")
        done += k
        st = state.cpu().numpy()                        # one host read per CG_CHECK_EVERY iterations
        for r in idx:
            if st[r, _native.AK_CG_BREAKDOWN_AT] > 0.0:
                msgs[r] = (f"p^T A p = {st[r, _native.AK_CG_BREAKDOWN_PAP]:.3e} <= 0 "
                           f"at iteration {int(st[r, _native.AK_CG_BREAKDOWN_AT])}")
                active[r] = False
            elif st[r, _native.AK_CG_ACTIVE] == 0.0:
                iters[r] = int(st[r, _native.AK_CG_ITERATIONS])
                active[r] = False
    for r in np.nonzero(active)[0]:
        msgs[r] = f"CG did not reach tol={tol} within {max_iter} iterations"
    return X, iters, msgs


def _grid_chunk(plan, R: int) -> int:
    """Cells per lockstep batch: the batched CG holds, per cell, the per-RHS operator's
    two grids and spectra (plus power-of-two bucket operators and the prediction
    operator, about 4 operator copies) and ~8 length-N vectors; use at most half of
    the free device memory (the reference runs one cell at a time)."""
    import torch

    free, _ = torch.cuda.mem_get_info()
    per_cell = 8 * (4 * 3 * plan.geometries.canon_total + 8 * plan.n_rows)
    return max(1, min(R, int(0.5 * free // max(per_cell, 1))))


def grid_search(train: Dataset, test: Dataset, ws: WindowSet, ell_grid, beta_grid, family: str = "gauss",
                backend: str = FASTSUM, preset="default", sigma_f: float | None = None,
                tol: float = DEFAULT_CG_TOL, max_iter: int = DEFAULT_CG_MAX_ITER) -> GridSearchResult:
    """Fit and score every (ell, beta) pair; ties favour small ell, beta (solver.py:157-198).

    ell values are in quarter-box units (rescaled by 1/sqrt(d_max) internally).
    With the fast-summation backend all cells run as one batched lockstep CG.
    """
    ell_grid = [float(e) for e in ell_grid]
    beta_grid = [float(b) for b in beta_grid]
    if not ell_grid or not beta_grid:
        raise ValueError("grids must be nonempty")
    if train.d_max is None:
        raise InvalidScalingError("training data must be prescaled")
    factor = 1.0 / math.sqrt(train.d_max)
    sf = default_sigma_f(len(ws)) if sigma_f is None else sigma_f
    pairs = [(e, b) for e in ell_grid for b in beta_grid]
    if backend != FASTSUM:
        return _grid_search_sequential(train, test, ws, pairs, family, backend, preset, sf, tol, max_iter, factor)

    import torch

    from .fastsum import build_plan, prepare_eval_points

    if train.scaling_state != PRESCALED:
        raise InvalidScalingError("krr_fit requires prescaled training data")
    if test.scaling_state != PRESCALED or not same_scaling(train, test):
        raise ScalingMismatchError("test data must be prescaled with the training maps")
    specs = [KernelSpec(family, e * factor, sf) for e, _ in pairs]
    t0 = time.perf_counter()
    with warnings.catch_warnings(record=True) as caught:
        warnings.simplefilter("always")
        plan = build_plan(specs[0], ws, preset, train)
        from .fastsum import _eta_warning

        for s in specs[1:]:
            _eta_warning(s.ell, plan.m)
    for w in caught:
        warnings.warn_explicit(w.message, w.category, w.filename, w.lineno)
    tp = time.perf_counter()
    R = len(pairs)
    chunk = _grid_chunk(plan, R)
    geoms = prepare_eval_points(plan, test)
    iters = np.zeros(R, dtype=np.int64)
    msgs = [None] * R
    pred_h = np.empty((R, test.n_rows))
    t_fit = t_pred = 0.0
    for c0 in range(0, R, chunk):
        # cells in batches sized to the free device memory (each batch: one lockstep CG)
        sl = slice(c0, min(R, c0 + chunk))
        cs, ps = specs[sl], pairs[sl]
        Rc = len(cs)
        ta = time.perf_counter()
        op = _grid_operator(plan, cs, Rc)
        apply_subset = _subset_applier(plan, cs, op)

        def apply(Pm, op=op):
            out = torch.empty_like(Pm)
            op.apply(Pm.contiguous(), [out], [True])
            return out

        Y = torch.as_tensor(np.broadcast_to(train.targets, (Rc, train.n_rows)).copy(), device="cuda")
        X, it_c, msg_c = cg_solve_batched(apply, Y, [b for _, b in ps], tol=tol, max_iter=max_iter,
                                          apply_subset=apply_subset)
        torch.cuda.synchronize()
        tb = time.perf_counter()
        del op, apply_subset, apply, Y
        pop = _grid_operator(plan, cs, Rc, interp_geom=geoms)
        pred = torch.empty((Rc, test.n_rows), dtype=torch.float64, device="cuda")
        pop.apply(X.contiguous(), [pred], [True])
        pred_h[sl] = pred.cpu().numpy()
        del pop, pred, X
        t_fit += tb - ta
        t_pred += time.perf_counter() - tb
        iters[sl] = it_c
        msgs[sl] = msg_c
    t1, t2 = tp + t_fit, tp + t_fit + t_pred   # plan build counted with the fits (t0 .. tp)
    cells = []
    for r, (e, b) in enumerate(pairs):
        if iters[r] < 0:
            cells.append(GridCell(e, b, None, None, (t1 - t0) / R, 0.0, failed=True, message=msgs[r]))
        else:
            cells.append(GridCell(e, b, rmse(test.targets, pred_h[r]), int(iters[r]), (t1 - t0) / R, (t2 - t1) / R))
    ok = [c for c in cells if not c.failed]
    if not ok:
        raise MaxIterationsError("every grid cell failed")
    best = min(ok, key=lambda c: (c.rmse, c.ell, c.beta))
    return GridSearchResult(cells=tuple(cells), best=best)


def _grid_search_sequential(train, test, ws, pairs, family, backend, preset, sf, tol, max_iter, factor):
    cells = []
    for e, b in pairs:
        spec = KernelSpec(family, e * factor, sf)
        t0 = time.perf_counter()
        try:
            model = krr_fit(train, ws, spec, b, backend=backend, preset=preset, tol=tol, max_iter=max_iter)
        except (MaxIterationsError, CgBreakdownError) as exc:
            cells.append(GridCell(e, b, None, None, time.perf_counter() - t0, 0.0, failed=True, message=str(exc)))
            continue
        t1 = time.perf_counter()
        pred = krr_predict(model, test)
        t2 = time.perf_counter()
        cells.append(GridCell(e, b, rmse(test.targets, pred), model.cg_iterations, t1 - t0, t2 - t1))
    ok = [c for c in cells if not c.failed]
    if not ok:
        raise MaxIterationsError("every grid cell failed")
    best = min(ok, key=lambda c: (c.rmse, c.ell, c.beta))
    return GridSearchResult(cells=tuple(cells), best=best)
