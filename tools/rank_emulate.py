"""Per-rank device time of the multi-GPU layouts, emulated on one GPU (no collectives).

For world sizes 2/4/8, every rank's share of config 4 (K v) is built and timed
alone: hybrid (window groups x row blocks, HybridShardedPlan) and cell slabs
(window groups x whole-cell slabs, CellShardedPlan).  The step of a real run is
the slowest rank plus the collectives (band all-reduce within a window group,
row all-reduce / all-gather of the 8 MB product), which are not included.

    python tools/rank_emulate.py [--worlds 2 4 8]
"""
import argparse
import json
import sys
from dataclasses import replace
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2404_17344_b200 import _native, configs  # noqa: E402
from paper_2404_17344_b200.distributed import cell_partition, hybrid_layout, row_partition, window_partition  # noqa: E402
from paper_2404_17344_b200.fastsum import build_plan  # noqa: E402
from paper_2404_17344_b200.windows import WindowSet  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--worlds", type=int, nargs="+", default=[2, 4, 8])
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--overheads", type=float, nargs="+", default=[0.0, 64.0, 256.0])
args = ap.parse_args()

wl = configs.config4()
ws, data, spec = wl.window_set, wl.data, wl.spec
V = torch.as_tensor(wl.V[:1], device="cuda")


def timed(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / args.reps


def hybrid_rank(world, rank):
    G = hybrid_layout(ws.lengths, world)
    Q = world // G
    owned = window_partition(ws.lengths, G)[rank // Q]
    lo, hi = row_partition(data.n_rows, Q)[rank % Q]
    sub = WindowSet(tuple(ws.windows[w] for w in owned), d_max=ws.d_max)
    plan = build_plan(spec, sub, "default", replace(data, features=data.features[lo:hi], targets=data.targets[lo:hi]))
    op = plan._operator((spec.family,), 1)
    Vl = V[:, lo:hi].contiguous()
    out = [torch.empty((1, hi - lo), dtype=torch.float64, device="cuda")]

    def step():
        op.spectrum_only(Vl)
        op.apply(None, out, [True], flags=_native.AK_APPLY_FROM_SPECTRUM)
    return timed(step)


def cell_rank(world, rank, G=None):
    G = G or hybrid_layout(ws.lengths, world)
    Q = world // G
    owned = window_partition(ws.lengths, G)[rank // Q]
    wins = tuple(ws.windows[w] for w in owned)
    masks = np.zeros((len(wins), data.n_rows), dtype=bool)
    for k, win in enumerate(wins):
        masks[k, cell_partition(data.features[:, list(ws.columns(win))], 64, Q, OVH)[rank % Q]] = True
    plan = build_plan(spec, WindowSet(wins, d_max=ws.d_max), "default", data, row_masks=masks)
    op = plan._operator((spec.family,), 1)
    out = [torch.empty((1, data.n_rows), dtype=torch.float64, device="cuda")]

    def step():
        op.spectrum_only(V)
        op.apply(None, out, [True], flags=_native.AK_APPLY_FROM_SPECTRUM)
    return timed(step)


plan1 = build_plan(spec, ws, "default", data)
op1 = plan1._operator((spec.family,), 1)
o1 = [torch.empty((1, data.n_rows), dtype=torch.float64, device="cuda")]
t1 = timed(lambda: op1.apply(V, o1, [True]))
res = {"single_gpu_ms": t1}
for world in args.worlds:
    h = [hybrid_rank(world, r) for r in range(world)]
    res[str(world)] = {"hybrid_max_ms": max(h), "ideal_ms": t1 / world, "hybrid_ranks": [round(x, 4) for x in h]}
    for OVH in args.overheads:
        c = [cell_rank(world, r) for r in range(world)]
        res[str(world)][f"cell_ovh{OVH:g}_max_ms"] = max(c)
        res[str(world)][f"cell_ovh{OVH:g}_ranks"] = [round(x, 4) for x in c]
    torch.cuda.empty_cache()
print(json.dumps(res))
