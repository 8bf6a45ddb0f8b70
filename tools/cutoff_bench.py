"""Config 4 with the non-default cutoff knob (build_plan(..., cutoff=c)): device time per
K v and the relative change of the result against the default cutoff 6."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2404_17344_b200 import configs  # noqa: E402
from paper_2404_17344_b200.fastsum import build_plan, fast_matvec  # noqa: E402

wl = configs.config4()
v = torch.as_tensor(wl.V[0], device="cuda")
ref = None
for c in (6, 5, 4, 3):
    plan = build_plan(wl.spec, wl.window_set, "default", wl.data, cutoff=c)
    out = fast_matvec(plan, v)
    ms = bench.cuda_time(torch, lambda: fast_matvec(plan, v), 10)
    if ref is None:
        ref = out.clone()
    err = float(torch.linalg.vector_norm(out - ref) / torch.linalg.vector_norm(ref))
    print(f"cutoff {c}: {ms:.3f} ms per K v, rel. change vs cutoff 6: {err:.2e}")
