"""Multi-GPU fast summation: one process per GPU, NCCL through torch.distributed.

The reference is single-process; its window loop
(fastsum.py:156-159) is a sum of independent per-window products, and each
window's product is linear in the spread grid, which gives two exact
decompositions:

* window sharding -- rank r owns a subset of the windows (longest-processing-
  time assignment by per-point cost T^q), computes sum_{w in own} K_w v for
  all N rows, and one all-reduce(sum) of the N x R products assembles K v on
  every rank.  Balance is capped by the window granularity (10 windows on 8
  GPUs: at most 5x).
* point sharding -- rank r owns a contiguous block of rows.  It spreads only
  its own nodes into every window's grid and transforms it; the band of the
  half spectra (R * sum_w m^(q-1) m/2 complex values: 2.6 MB for config 4,
  8x less than the 20 MB of grids) is summed with one all-reduce, every rank
  runs the multiply / inverse FFT redundantly and interpolates only its own
  rows.  The spread and the FFT are linear, so the summed band equals the band
  of the summed grid.  The result is row-sharded (all_gather for a replicated
  vector).  Balanced for any window mix.  ``exchange="grid"`` all-reduces the
  grids instead (before the FFT).

HybridShardedPlan combines them (window groups x row blocks); CellShardedPlan
(the bench default) uses window groups x slabs of whole grid cells, so every
rank keeps the data's full per-cell density.  All reproduce the single-GPU
product up to the order of floating-point sums.
"""

from __future__ import annotations

import heapq

from .dataset import Dataset
from .windows import WindowSet

WINDOW_TAPS = 12
#: per-cell cost of a work item (prologue + register-tile flush) in row equivalents,
#: for balancing cell slabs (tools/rank_emulate.py)
CELL_OVERHEAD_ROWS = 64.0


def window_cost(q: int, taps: int = WINDOW_TAPS) -> int:
    """Per-point spread + interp cost of a window of length q (FMAs ~ taps^q)."""
    return taps ** q


def window_partition(lengths, world: int, taps: int = WINDOW_TAPS) -> list:
    """Assign windows to ranks, longest-processing-time first (greedy LPT).

    Returns world lists of window indices (ascending); ranks may be empty when
    there are fewer windows than ranks.
    """
    order = sorted(range(len(lengths)), key=lambda w: (-window_cost(lengths[w], taps), w))
    heap = [(0, r) for r in range(world)]
    owned = [[] for _ in range(world)]
    for w in order:
        load, r = heapq.heappop(heap)
        owned[r].append(w)
        heapq.heappush(heap, (load + window_cost(lengths[w], taps), r))
    return [sorted(o) for o in owned]


def row_partition(n_rows: int, world: int) -> list:
    """Contiguous, balanced row blocks [(lo, hi), ...] for point sharding."""
    base, extra = divmod(n_rows, world)
    out, lo = [], 0
    for r in range(world):
        hi = lo + base + (1 if r < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


def _dist():
    import torch.distributed as dist

    return dist


_GROUPS: dict = {}
_GROUPS_WORLD = [None]   # the default group the cache belongs to (re-initialised: cache dropped)


def _new_group(members):
    """dist.new_group, cached per member list: plans rebuilt under one process group
    (a grid search, repeated hyperparameters) reuse the communicators instead of
    creating new ones every time.  Like new_group itself, every rank must call it for
    every group, in the same order."""
    dist = _dist()
    if _GROUPS_WORLD[0] is not dist.group.WORLD:
        _GROUPS.clear()
        _GROUPS_WORLD[0] = dist.group.WORLD
    key = tuple(members)
    pg = _GROUPS.get(key)
    if pg is None:
        pg = dist.new_group(list(members))
        _GROUPS[key] = pg
    return pg


class _StageClock:
    """Optional per-stage device timing of a sharded product (CUDA events on the
    current stream, collectives included): `profile(fn, steps)` returns the mean ms
    per step of each stage."""

    def __init__(self):
        self.on = False
        self.events = []

    def mark(self, name):
        if not self.on:
            return
        import torch

        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        self.events.append((name, ev))

    def profile(self, fn, steps: int) -> dict:
        import torch

        self.on, self.events = True, []
        torch.cuda.synchronize()
        for _ in range(steps):
            self.mark("start")
            fn()
            self.mark("end")
        torch.cuda.synchronize()
        self.on = False
        out = {}
        for (_, a), (name, b) in zip(self.events[:-1], self.events[1:]):
            if name == "start":
                continue
            key = "other" if name == "end" else name   # after the last stage: result assembly
            out[key] = out.get(key, 0.0) + a.elapsed_time(b) / steps
        self.events = []
        return out


def _default_builder():
    from .fastsum import build_plan

    return build_plan


def _subset_rows(data: Dataset, lo: int, hi: int) -> Dataset:
    from dataclasses import replace

    return replace(data, features=data.features[lo:hi], targets=data.targets[lo:hi])


class WindowShardedPlan:
    """K v over all windows with the windows split across ranks."""

    def __init__(self, spec, window_set: WindowSet, preset, data: Dataset, group=None, plan_builder=None, **kw):
        dist = _dist()
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.spec = spec
        self.owned = window_partition(window_set.lengths, self.world)[self.rank]
        self.n_rows = data.n_rows
        self.plan = None
        self.clock = _StageClock()
        if self.owned:   # ranks beyond the window count own nothing and contribute zeros
            sub = WindowSet(tuple(window_set.windows[w] for w in self.owned), d_max=window_set.d_max)
            self.plan = (plan_builder or _default_builder())(spec, sub, preset, data, **kw)

    def matvecs(self, V, families=None):
        """(R, N) tensor -> list of (R, N) products (one per coefficient set), replicated."""
        import torch

        dist = _dist()
        fams = tuple(families or (self.spec.family,))
        R = V.shape[0]
        outs = [torch.zeros((R, self.n_rows), dtype=torch.float64, device=V.device) for _ in fams]
        if self.plan is not None:
            self.plan._operator(fams, R).apply(V, outs, [True] * len(outs))
        self.clock.mark("windows")
        for o in outs:
            dist.all_reduce(o, group=self.group)
        self.clock.mark("allreduce_rows")
        return outs

    def stage_times(self, fn, steps: int = 5) -> dict:
        return self.clock.profile(fn, steps)

    def matvec(self, v):
        return self.matvecs(v.reshape(1, -1))[0][0]


class PointShardedPlan:
    """K v with the rows split across ranks; band spectra (or grids) are all-reduced."""

    def __init__(self, spec, window_set: WindowSet, preset, data: Dataset, group=None, exchange: str = "band",
                 **kw):
        from .fastsum import build_plan

        if exchange not in ("band", "grid"):
            raise ValueError("exchange must be 'band' or 'grid'")
        dist = _dist()
        self.exchange = exchange
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.rows = row_partition(data.n_rows, self.world)
        self.lo, self.hi = self.rows[self.rank]
        self.n_rows = data.n_rows
        self.plan = build_plan(spec, window_set, preset, _subset_rows(data, self.lo, self.hi), **kw)

    def matvecs_local(self, V_local, families=None):
        """(R, n_local) own-row RHS block -> list of (R, n_local) own-row products."""
        import torch

        dist = _dist()
        fams = tuple(families or (self.plan.spec.family,))
        R = V_local.shape[0]
        from . import _native

        op = self.plan._operator(fams, R)
        if self.exchange == "band":
            op.spectrum_only(V_local)
            dist.all_reduce(op.band(), group=self.group)
            flag = _native.AK_APPLY_FROM_SPECTRUM
        else:
            op.spread_only(V_local)
            dist.all_reduce(op.grids(), group=self.group)
            flag = _native.AK_APPLY_FROM_GRIDS
        outs = [torch.empty((R, self.hi - self.lo), dtype=torch.float64, device="cuda") for _ in fams]
        op.apply(None, outs, [True] * len(outs), flags=flag)
        return outs

    def matvec(self, v, gather: bool = True):
        """Full-length v (replicated) -> K v (replicated if gather, else own rows)."""
        import torch

        dist = _dist()
        out = self.matvecs_local(v[self.lo:self.hi].reshape(1, -1))[0][0]
        if not gather:
            return out
        sizes = [hi - lo for lo, hi in self.rows]
        chunks = [torch.empty(s, dtype=torch.float64, device="cuda") for s in sizes]
        if len(set(sizes)) == 1:
            dist.all_gather(chunks, out, group=self.group)
        else:
            m = max(sizes)
            pad = torch.zeros(m, dtype=torch.float64, device="cuda")
            pad[: out.numel()] = out
            bufs = [torch.empty(m, dtype=torch.float64, device="cuda") for _ in sizes]
            dist.all_gather(bufs, pad, group=self.group)
            chunks = [b[:s] for b, s in zip(bufs, sizes)]
        return torch.cat(chunks)


def hybrid_layout(lengths, world: int, taps: int = WINDOW_TAPS, tolerance: float = 0.1) -> int:
    """Number of window groups for HybridShardedPlan: the largest g in {world, ..., 2}
    dividing world whose LPT window partition is balanced within `tolerance`
    (max group cost <= (1 + tolerance) * mean), else 1 (pure point sharding)."""
    total = sum(window_cost(q, taps) for q in lengths)
    for g in range(min(world, len(lengths)), 1, -1):
        if world % g:
            continue
        parts = window_partition(lengths, g, taps)
        worst = max(sum(window_cost(lengths[w], taps) for w in p) for p in parts)
        if worst <= (1.0 + tolerance) * total / g:
            return g
    return 1


class HybridShardedPlan:
    """Window groups x point groups (the two exact decompositions combined).

    world = G x Q ranks: window group gi = rank // Q owns an LPT share of the
    windows, point group position pj = rank % Q owns a contiguous row block.
    Each rank spreads its rows into its windows' grids; the band spectra are
    all-reduced among the Q ranks of its window group; each rank interpolates
    its own rows for its own windows; the partial products of a row block are
    all-reduced across the G window groups.  G = 1 is point sharding, Q = 1 is
    window sharding.  Per rank: 1/world of the gridding work and 1/G of the
    FFTs (point sharding repeats all FFTs on every rank), with one small
    collective per stage: band (R * sum_w m^(q-1) m/2 complex over own
    windows) and rows (R * N/Q doubles).
    """

    def __init__(self, spec, window_set: WindowSet, preset, data: Dataset, window_groups: int | None = None,
                 group=None, **kw):
        from .fastsum import build_plan

        dist = _dist()
        world = dist.get_world_size(group)
        rank = dist.get_rank(group)
        G = window_groups or hybrid_layout(window_set.lengths, world)
        if G < 1 or world % G or G > len(window_set):
            raise ValueError("window_groups must divide the world size and not exceed the number of windows")
        Q = world // G
        self.world, self.rank, self.G, self.Q = world, rank, G, Q
        self.gi, self.pj = rank // Q, rank % Q
        base = dist.get_process_group_ranks(group) if group is not None else list(range(world))
        # every rank creates every subgroup (new_group is collective)
        self.band_group = self.row_group = None
        for g in range(G):
            members = [base[g * Q + j] for j in range(Q)]
            pg = _new_group(members) if Q > 1 else None
            if g == self.gi:
                self.band_group = pg
        for j in range(Q):
            members = [base[g * Q + j] for g in range(G)]
            pg = _new_group(members) if G > 1 else None
            if j == self.pj:
                self.row_group = pg
        self.owned = window_partition(window_set.lengths, G)[self.gi]
        self.rows = row_partition(data.n_rows, Q)
        self.lo, self.hi = self.rows[self.pj]
        self.n_rows = data.n_rows
        sub = WindowSet(tuple(window_set.windows[w] for w in self.owned), d_max=window_set.d_max)
        self.plan = build_plan(spec, sub, preset, _subset_rows(data, self.lo, self.hi), **kw)

    def matvecs_local(self, V_local, families=None):
        """(R, n_local) own-row RHS block -> list of (R, n_local) own-row products (all windows)."""
        import torch

        from . import _native

        dist = _dist()
        fams = tuple(families or (self.plan.spec.family,))
        R = V_local.shape[0]
        op = self.plan._operator(fams, R)
        if self.Q > 1:
            op.spectrum_only(V_local)
            dist.all_reduce(op.band(), group=self.band_group)
            flag = _native.AK_APPLY_FROM_SPECTRUM
            V_arg = None
        else:
            flag, V_arg = 0, V_local
        outs = [torch.empty((R, self.hi - self.lo), dtype=torch.float64, device="cuda") for _ in fams]
        op.apply(V_arg, outs, [True] * len(outs), flags=flag)
        if self.G > 1:
            for o in outs:
                dist.all_reduce(o, group=self.row_group)
        return outs

    def matvec(self, v, gather: bool = True):
        """Full-length v (replicated) -> K v (replicated if gather, else own rows)."""
        import torch

        dist = _dist()
        out = self.matvecs_local(v[self.lo:self.hi].reshape(1, -1))[0][0]
        if not gather:
            return out
        if self.Q == 1:
            return out
        sizes = [hi - lo for lo, hi in self.rows]
        m = max(sizes)
        pad = torch.zeros(m, dtype=torch.float64, device="cuda")
        pad[: out.numel()] = out
        bufs = [torch.empty(m, dtype=torch.float64, device="cuda") for _ in sizes]
        dist.all_gather(bufs, pad, group=self.band_group)
        return torch.cat([b[:s] for b, s in zip(bufs, sizes)])


def cell_partition(coords, n: int, parts: int, cell_overhead: float = 0.0) -> list:
    """Split the rows of one window into `parts` sets of whole grid cells.

    coords: (N, q) prescaled window coordinates in [-1/2, 1/2).  A row's cell is
    floor((x + 1/2) n) per axis (the cell whose footprint it spreads into,
    nufft.py:183-186); cells are ordered by linear index (slabs along the first
    axis) and cut into `parts` contiguous runs of balanced cost, a cell costing
    its row count plus `cell_overhead` (per-cell work item prologue and flush,
    in row equivalents).
    Returns `parts` ascending int64 row-index arrays (some may be empty when
    there are fewer occupied cells than parts).
    """
    import numpy as np

    coords = np.asarray(coords, dtype=np.float64)
    if coords.ndim == 1:
        coords = coords[:, None]
    t = np.clip(np.floor((coords + 0.5) * n).astype(np.int64), 0, n - 1)
    lin = np.zeros(coords.shape[0], dtype=np.int64)
    for a in range(coords.shape[1]):
        lin = lin * n + t[:, a]
    order = np.argsort(lin, kind="stable")
    cells, starts, counts = np.unique(lin[order], return_index=True, return_counts=True)
    cum = np.cumsum(counts + cell_overhead)
    total = int(cum[-1]) if len(cum) else 0
    # cell run p ends at the first cell whose cumulative count reaches (p + 1) / parts
    bounds = [0]
    for p in range(1, parts):
        bounds.append(int(np.searchsorted(cum, total * p / parts, side="left")) + 1 if total else 0)
    bounds.append(len(cells))
    bounds = np.maximum.accumulate(np.minimum(np.array(bounds), len(cells)))
    edges = np.append(starts, coords.shape[0])   # row offset of each cell run in `order`
    return [np.sort(order[edges[bounds[p]]:edges[bounds[p + 1]]]).astype(np.int64) for p in range(parts)]


class CellShardedPlan:
    """Window groups x cell slabs: the hybrid layout with each window's rows split
    by grid cell instead of by row block.

    world = G x Q ranks as in HybridShardedPlan.  Within a window group every
    owned window's occupied cells are cut into Q slabs of equal row count
    (cell_partition), so each rank spreads and interpolates whole cells at the
    data's full density (the single-cell kernels keep their efficiency, where a
    row block of N/Q rows thins every cell Q-fold).  The rank holds ONE plan over
    its owned windows with a per-window row mask (build_plan(row_masks=...),
    ak_geom_create_masked): one spread / transform / interpolation launch for all
    of them, outputs indexed by the global rows.  The band spectra are
    all-reduced among the Q ranks of the group; one all-reduce over all ranks of
    the length-N partial products assembles K v on every rank.
    """

    def __init__(self, spec, window_set: WindowSet, preset, data: Dataset, window_groups: int | None = None,
                 group=None, plan_builder=None, **kw):
        import numpy as np

        from .fastsum import resolve_m
        from .nufft import NufftPlan

        dist = _dist()
        world = dist.get_world_size(group)
        rank = dist.get_rank(group)
        G = window_groups or hybrid_layout(window_set.lengths, world)
        if G < 1 or world % G or G > len(window_set):
            raise ValueError("window_groups must divide the world size and not exceed the number of windows")
        Q = world // G
        self.world, self.rank, self.G, self.Q, self.group = world, rank, G, Q, group
        self.gi, self.pj = rank // Q, rank % Q
        base = dist.get_process_group_ranks(group) if group is not None else list(range(world))
        self.band_group = None
        for g in range(G):
            members = [base[g * Q + j] for j in range(Q)]
            pg = _new_group(members) if Q > 1 else None
            if g == self.gi:
                self.band_group = pg
        self.owned = window_partition(window_set.lengths, G)[self.gi]
        self.n_rows = data.n_rows
        self.spec = spec
        self.clock = _StageClock()
        m = resolve_m(preset)
        wins = tuple(window_set.windows[w] for w in self.owned)
        masks = np.zeros((len(wins), data.n_rows), dtype=bool)
        for k, win in enumerate(wins):
            n = NufftPlan(dims=len(win), m=m, cutoff=kw.get("cutoff", 6),
                          oversampling=kw.get("oversampling", 2.0)).n
            masks[k, cell_partition(data.features[:, list(window_set.columns(win))], n, Q,
                                    CELL_OVERHEAD_ROWS)[self.pj]] = True
        self.rows_per_window = masks.sum(axis=1)
        self.plan = (plan_builder or _default_builder())(spec, WindowSet(wins, d_max=window_set.d_max), preset, data,
                                                         row_masks=masks, **kw)

    def matvecs(self, V, families=None):
        """(R, N) replicated RHS -> list of (R, N) replicated products (one per family)."""
        import torch

        from . import _native

        dist = _dist()
        fams = tuple(families or (self.spec.family,))
        R = V.shape[0]
        outs = [torch.empty((R, self.n_rows), dtype=torch.float64, device=V.device) for _ in fams]
        op = self.plan._operator(fams, R)
        if self.Q > 1:
            op.spectrum_only(V)
            self.clock.mark("spread_fwd_transform")
            dist.all_reduce(op.band(), group=self.band_group)
            self.clock.mark("allreduce_band")
            op.apply(None, outs, [True] * len(outs), flags=_native.AK_APPLY_FROM_SPECTRUM)
            self.clock.mark("multiply_inverse_interp")
        else:
            op.apply(V, outs, [True] * len(outs))
            self.clock.mark("windows")
        if self.world > 1:
            for o in outs:
                dist.all_reduce(o, group=self.group)
            self.clock.mark("allreduce_rows")
        return outs

    def stage_times(self, fn, steps: int = 5) -> dict:
        return self.clock.profile(fn, steps)

    def matvec(self, v):
        """Full-length v (replicated) -> K v (replicated)."""
        return self.matvecs(v.reshape(1, -1))[0][0]
