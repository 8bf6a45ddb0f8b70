"""krr_fit (CG on the GPU operator) per-iteration cost vs the product alone."""
import math
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2404_17344_b200.dataset import PRESCALED, Dataset  # noqa: E402
from paper_2404_17344_b200.fastsum import build_plan, fast_matvec  # noqa: E402
from paper_2404_17344_b200.kernels import KernelSpec  # noqa: E402
from paper_2404_17344_b200.solver import default_sigma_f, krr_fit  # noqa: E402
from paper_2404_17344_b200.windows import WindowSet  # noqa: E402

for n in (20_000, 100_000):
    rng = np.random.default_rng(3)
    X = rng.uniform(-0.25, 0.25, size=(n, 9)) / np.sqrt(3)
    y = np.sin(8 * X[:, 0]) + np.cos(6 * X[:, 4] * X[:, 5]) + 0.1 * rng.normal(size=n)
    tr = Dataset(X, y, tuple(f"x{i + 1}" for i in range(9)), scaling_state=PRESCALED, d_max=3)
    ws = WindowSet(((1, 2, 3), (4, 5, 6), (7, 8, 9)), d_max=3)
    spec = KernelSpec("gauss", 0.2 / math.sqrt(3), default_sigma_f(3))
    krr_fit(tr, ws, spec, 0.1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    m = krr_fit(tr, ws, spec, 0.1)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    plan = build_plan(spec, ws, "default", tr)
    v = torch.as_tensor(y, device="cuda")
    fast_matvec(plan, v)  # operator + cuFFT plans created outside the timing
    ms = bench.cuda_time(torch, lambda: fast_matvec(plan, v), 20)
    print(f"N={n}: krr_fit {dt * 1e3:.1f} ms for {m.cg_iterations} CG iterations "
          f"({dt * 1e3 / max(1, m.cg_iterations):.3f} ms/iteration incl. plan build); product alone {ms:.3f} ms")
