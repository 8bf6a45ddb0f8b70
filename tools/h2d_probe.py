"""H2D of an 8 MB pageable numpy vector: driver-staged copy vs threaded pinned staging.

Measured on the B200 box (16 vCPUs): pageable 0.43 ms, best threaded staging 0.26 ms
in Python, but a C++ staging pool with overlapped slice DMAs lost (0.5-1.4 ms): host
memory bandwidth (~35-45 GB/s aggregate, tools/memcpy_probe.cu) is shared by the
staging copies and the DMA reads, so the driver path stays."""
import sys, time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch, os
N = 1_000_000
v = np.random.default_rng(0).normal(size=N)
d = torch.empty(N, dtype=torch.float64, device="cuda")
pin = torch.empty(N, dtype=torch.float64, pin_memory=True)
pn = pin.numpy()
print("cpus", os.cpu_count(), len(os.sched_getaffinity(0)))
def t(fn, reps=50):
    for _ in range(3): fn()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps * 1e3
print("pageable .to/copy_  ms", t(lambda: d.copy_(torch.from_numpy(v))))
print("memcpy to pinned    ms", t(lambda: np.copyto(pn, v)))
print("pinned H2D only     ms", t(lambda: d.copy_(pin, non_blocking=True)))
for nt in (2, 4, 8, 16):
    pool = ThreadPoolExecutor(nt)
    def staged(nt=nt, pool=pool):
        b = np.linspace(0, N, nt + 1).astype(int)
        futs = [pool.submit(np.copyto, pn[b[i]:b[i+1]], v[b[i]:b[i+1]]) for i in range(nt)]
        for f in futs: f.result()
        d.copy_(pin, non_blocking=True)
    print(f"threaded({nt}) stage+H2D ms", t(staged))
    def piped(nt=nt, pool=pool):
        b = np.linspace(0, N, nt + 1).astype(int)
        futs = [pool.submit(np.copyto, pn[b[i]:b[i+1]], v[b[i]:b[i+1]]) for i in range(nt)]
        for i, f in enumerate(futs):
            f.result()
            d[b[i]:b[i+1]].copy_(pin[b[i]:b[i+1]], non_blocking=True)
    print(f"threaded({nt}) piped     ms", t(piped))
host = torch.empty(N, dtype=torch.float64, pin_memory=True)
def d2h():
    host.copy_(d, non_blocking=True); torch.cuda.current_stream().synchronize()
print("d2h pinned          ms", t(d2h))
