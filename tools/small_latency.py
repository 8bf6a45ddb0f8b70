"""Per-product latency at small N (configs 1-3): device events vs wall clock per call."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2404_17344_b200 import _native, configs  # noqa: E402
from paper_2404_17344_b200.fastsum import build_plan, fast_matvec  # noqa: E402

for name in ("C1", "C2", "C3"):
    wl = configs.CONFIGS[name]()
    plan = build_plan(wl.spec, wl.window_set, "default", wl.data)
    v = torch.as_tensor(wl.V[0], device="cuda")
    for _ in range(5):
        fast_matvec(plan, v)
    torch.cuda.synchronize()
    reps = 200
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = _native.launch_count()
    t0 = time.perf_counter()
    e0.record()
    for _ in range(reps):
        fast_matvec(plan, v)
    e1.record()
    e1.synchronize()
    wall = (time.perf_counter() - t0) / reps * 1e3
    t1 = time.perf_counter()
    for _ in range(reps):
        fast_matvec(plan, v)
        torch.cuda.synchronize()
    sync = (time.perf_counter() - t1) / reps * 1e3
    print(f"{name}: N={wl.data.n_rows} events {e0.elapsed_time(e1) / reps:.4f} ms, wall (pipelined) {wall:.4f} ms, "
          f"wall (sync each) {sync:.4f} ms, launches/product {(_native.launch_count() - l0) / reps:.1f}")
