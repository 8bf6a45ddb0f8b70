"""Do the q=3 spread (DFMA) and interpolation (DMMA) kernels overlap profitably?
Measured on B200: sequential 2.90 ms, two streams 2.89 ms, and one fused launch
alternating spread / interpolation CTAs (so every SM runs both) 2.92 ms: the
two kernels share the FP64 datapath, co-residency raises nothing.
Config 4 geometry: ak_spread on one stream and ak_interp on another (independent
buffers), sequential vs concurrent, device time of the pair."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2404_17344_b200 import _native, configs  # noqa: E402
from paper_2404_17344_b200.fastsum import build_plan  # noqa: E402

wl = configs.config4()
plan = build_plan(wl.spec, wl.window_set, "default", wl.data)
lib = _native.lib()
geom = plan.geometries
N = wl.data.n_rows
V = torch.as_tensor(wl.V[:1], device="cuda").contiguous()
gA = torch.zeros(geom.canon_total, dtype=torch.float64, device="cuda")
gB = torch.randn(geom.canon_total, dtype=torch.float64, device="cuda")
out = torch.zeros(N, dtype=torch.float64, device="cuda")
scale = torch.ones(geom.n_windows, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def spread(st):
    _native.check(lib.ak_spread(geom.handle, V.data_ptr(), 1, N, gA.data_ptr(), st.cuda_stream))


def interp(st):
    _native.check(lib.ak_interp(geom.handle, gB.data_ptr(), 1, scale.data_ptr(), out.data_ptr(), N, 1, 0,
                                st.cuda_stream))


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


cur = torch.cuda.current_stream()


def seq():
    spread(cur)
    interp(cur)


def conc():
    ev = torch.cuda.Event()
    ev.record(cur)
    s1.wait_event(ev)
    s2.wait_event(ev)
    spread(s1)
    interp(s2)
    e1, e2 = torch.cuda.Event(), torch.cuda.Event()
    e1.record(s1)
    e2.record(s2)
    cur.wait_event(e1)
    cur.wait_event(e2)


print("spread alone  ms", timed(lambda: spread(cur)))
print("interp alone  ms", timed(lambda: interp(cur)))
print("sequential    ms", timed(seq))
print("concurrent    ms", timed(conc))

