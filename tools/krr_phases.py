"""Where krr_fit's wall time goes (plan build, graph capture, CG iterations, result copy)."""
import math
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2404_17344_b200 import solver  # noqa: E402
from paper_2404_17344_b200.dataset import PRESCALED, Dataset  # noqa: E402
from paper_2404_17344_b200.fastsum import build_plan, fast_matvec  # noqa: E402
from paper_2404_17344_b200.kernels import KernelSpec  # noqa: E402
from paper_2404_17344_b200.windows import WindowSet  # noqa: E402


def tick():
    torch.cuda.synchronize()
    return time.perf_counter()


for n in (20_000, 100_000, 1_000_000):
    rng = np.random.default_rng(3)
    X = rng.uniform(-0.25, 0.25, size=(n, 9)) / np.sqrt(3)
    y = np.sin(8 * X[:, 0]) + np.cos(6 * X[:, 4] * X[:, 5]) + 0.1 * rng.normal(size=n)
    tr = Dataset(X, y, tuple(f"x{i + 1}" for i in range(9)), scaling_state=PRESCALED, d_max=3)
    ws = WindowSet(((1, 2, 3), (4, 5, 6), (7, 8, 9)), d_max=3)
    spec = KernelSpec("gauss", 0.2 / math.sqrt(3), solver.default_sigma_f(3))
    plan = build_plan(spec, ws, "default", tr)
    yd = torch.as_tensor(tr.targets, device="cuda")
    mv = lambda p: fast_matvec(plan, p)  # noqa: E731
    fast_matvec(plan, yd)
    t0 = tick()
    for _ in range(50):
        fast_matvec(plan, yd)
    prod = (tick() - t0) / 50

    def per_iteration(fn):
        """Fixed iteration counts (tolerance 0): the difference of two caps is the per-iteration cost."""
        out = []
        for cap in (100, 1100):
            best = 1e9
            for _ in range(3):
                t0 = tick()
                try:
                    fn(cap)
                except solver.MaxIterationsError:
                    pass
                best = min(best, tick() - t0)
            out.append(best)
        return (out[1] - out[0]) / 1000, out[0] - 100 * (out[1] - out[0]) / 1000

    res = {}
    solver.CG_GRAPH_AFTER = 0
    for every in (1, 8):
        solver.CG_CHECK_EVERY = every
        res[f"graphed/{every}"] = per_iteration(lambda cap: solver._cg_solve_graphed(mv, yd, 0.1, 0.0, cap, None))
    solver.GRAPHED_CG = False
    for every in (1, 8):
        solver.CG_CHECK_EVERY = every
        res[f"native eager/{every}"] = per_iteration(lambda cap: solver._cg_solve_graphed(mv, yd, 0.1, 0.0, cap, None))
    solver.GRAPHED_CG, solver.CG_GRAPH_AFTER, solver.CG_CHECK_EVERY = True, 256, 8
    res["default (eager 256, then graph)"] = per_iteration(lambda cap: solver._cg_solve_graphed(mv, yd, 0.1, 0.0, cap, None))
    res["eager torch"] = per_iteration(lambda cap: solver._cg_solve_device(mv, yd, 0.1, 0.0, cap, None))
    print(f"N={n}: product {1e3 * prod:.3f} ms; " + "; ".join(f"{k}: {1e3 * a:.3f} ms/it (+{1e3 * b:.1f} ms setup)" for k, (a, b) in res.items()))
