"""H2D/D2H path costs for an 8 MB vector (pageable vs pinned)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
N = 1_000_000
v = np.random.default_rng(0).normal(size=N)
d = torch.empty(N, dtype=torch.float64, device="cuda")
def t(fn, reps=20):
    fn(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps * 1e3
print("h2d pageable   ms", t(lambda: d.copy_(torch.from_numpy(v))))
print("h2d pin+async  ms", t(lambda: d.copy_(torch.from_numpy(v).pin_memory(), non_blocking=True)))
print("d2h pageable   ms", t(lambda: d.cpu().numpy()))
def pin():
    h = torch.empty(N, dtype=torch.float64, pin_memory=True); h.copy_(d, non_blocking=True); torch.cuda.current_stream().synchronize(); return h.numpy()
print("d2h pinned     ms", t(pin))
