"""Grid search (tools/grid_search_bench.py's problem): wall time vs the library's kernel time."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2404_17344_b200 import _native  # noqa: E402
from paper_2404_17344_b200.dataset import PRESCALED, Dataset  # noqa: E402
from paper_2404_17344_b200.solver import grid_search  # noqa: E402
from paper_2404_17344_b200.windows import WindowSet  # noqa: E402

rng = np.random.default_rng(3)
n_tr, n_te, d = 20000, 4000, 9
X = rng.uniform(-0.25, 0.25, size=(n_tr + n_te, d)) / np.sqrt(3)
y = np.sin(8 * X[:, 0]) + np.cos(6 * X[:, 4] * X[:, 5]) + 0.1 * rng.normal(size=n_tr + n_te)
names = tuple(f"x{i + 1}" for i in range(d))
tr = Dataset(X[:n_tr], y[:n_tr], names, scaling_state=PRESCALED, d_max=3)
te = Dataset(X[n_tr:], y[n_tr:], names, scaling_state=PRESCALED, d_max=3)
ws = WindowSet(((1, 2, 3), (4, 5, 6), (7, 8, 9)), d_max=3)
ells, betas = [0.05, 0.1, 0.2, 0.3, 0.4], [1e-2, 1e-1, 1.0, 3.0, 10.0]
grid_search(tr, te, ws, ells, betas)
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = grid_search(tr, te, ws, ells, betas)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
with _native.KernelTimer() as kt:
    grid_search(tr, te, ws, ells, betas)
lib_ms = sum(ms for _, ms in kt.report.values())
its = [c.cg_iterations for c in res.cells if not c.failed]
print(f"25-cell grid search: {1e3 * dt:.1f} ms wall; library kernels {lib_ms:.1f} ms "
      f"({sum(n for n, _ in kt.report.values())} launches); CG iterations max {max(its)}, sum {sum(its)}")
