"""Kernel efficiency with negligible per-item overhead: 1M nodes packed into a few
cells (every work item holds the 2048-point cap) vs config 4 (items average ~370)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2404_17344_b200 import configs  # noqa: E402
from paper_2404_17344_b200.dataset import PRESCALED, Dataset  # noqa: E402
from paper_2404_17344_b200.fastsum import build_plan  # noqa: E402

wl = configs.config4()
rng = np.random.default_rng(0)
X = rng.uniform(-0.005, 0.005, size=wl.data.features.shape)
blob = configs.Workload("blob", Dataset(X, np.zeros(X.shape[0]), wl.data.feature_names, scaling_state=PRESCALED,
                                        d_max=3), wl.window_set, wl.specs, wl.V, False, False, False)
peaks = {"fp64_tflops": 36.7, "hbm_gbs": 6553.3}
for w in (wl, blob):
    plan = build_plan(w.spec, w.window_set, "default", w.data)
    r = bench.kernel_roofline(torch, plan, w, peaks, reps=20)
    print(f"{w.name}: items {plan.geometries.n_items}, spread {r['spread_ms']:.3f} ms "
          f"({r['flops_per_launch'] / (r['spread_ms'] * 1e-3) / 36.7e12:.1%}), interp {r['interp_ms']:.3f} ms "
          f"({r['flops_per_launch'] / (r['interp_ms'] * 1e-3) / 36.7e12:.1%})")
