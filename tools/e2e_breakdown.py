"""Where the e2e time goes (config 4): wall-clock per call of fast_matvec with a
device vector vs a host vector, device-event time, and the bare copies."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2404_17344_b200 import configs  # noqa: E402
from paper_2404_17344_b200.fastsum import build_plan, fast_matvec  # noqa: E402

wl = configs.config4()
plan = build_plan(wl.spec, wl.window_set, "default", wl.data)
v = np.ascontiguousarray(wl.V[0])
vd = torch.as_tensor(v, device="cuda")


def wall(fn, reps=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


def ev(fn, reps=30):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


def dev_sync():
    fast_matvec(plan, vd)
    torch.cuda.synchronize()


out = torch.empty(wl.data.n_rows, dtype=torch.float64, device="cuda")
host = torch.empty(wl.data.n_rows, dtype=torch.float64, pin_memory=True)
print("device events, device v      ms", ev(lambda: fast_matvec(plan, vd)))
print("wall, device v, sync per call ms", wall(dev_sync))
print("wall, host v -> numpy         ms", wall(lambda: fast_matvec(plan, v)))
print("wall, H2D pageable 8 MB       ms", wall(lambda: vd.copy_(torch.from_numpy(v))))
print("wall, D2H pinned 8 MB + sync  ms", wall(lambda: (host.copy_(out, non_blocking=True), torch.cuda.synchronize())))
