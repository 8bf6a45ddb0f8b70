"""Per-call latency of fast_matvec (device vector) for configs 1-4."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2404_17344_b200 import configs
from paper_2404_17344_b200.fastsum import build_plan, fast_matvec
for name in ("C1", "C2", "C3", "C4"):
    wl = configs.CONFIGS[name]()
    plan = build_plan(wl.spec, wl.window_set, "default", wl.data)
    v = torch.as_tensor(wl.V[0], device="cuda")
    for _ in range(3): fast_matvec(plan, v)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(50): fast_matvec(plan, v)
    torch.cuda.synchronize(); wall = (time.perf_counter() - t0) / 50 * 1e3
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(50): fast_matvec(plan, v)
    e1.record(); e1.synchronize()
    print(f"{name} N={wl.data.n_rows} windows={len(wl.window_set)} wall {wall:.3f} ms/call  device {e0.elapsed_time(e1)/50:.3f} ms/call")
