"""H2D of an 8 MB pageable numpy vector: cudaHostRegister in place."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
N = 1_000_000
d = torch.empty(N, dtype=torch.float64, device="cuda")
cr = torch.cuda.cudart()
def t(fn, reps=50):
    for _ in range(3): fn()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps * 1e3
vs = [np.random.default_rng(i).normal(size=N) for i in range(60)]
it = iter(range(10**9))
def reg():
    v = vs[next(it) % 60]
    p = v.ctypes.data
    cr.cudaHostRegister(p, v.nbytes, 0)
    d.copy_(torch.from_numpy(v), non_blocking=True)
    torch.cuda.current_stream().synchronize()
    cr.cudaHostUnregister(p)
print("register+H2D+unregister ms", t(reg))
def page():
    v = vs[next(it) % 60]
    d.copy_(torch.from_numpy(v))
print("pageable (fresh arrays)  ms", t(page))
