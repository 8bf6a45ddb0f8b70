"""The product's multi-GPU classes (distributed.WindowShardedPlan, CellShardedPlan)
run on CPU ranks (gloo, world sizes 2-4) with an oracle-backed stand-in for the
per-rank CUDA plan: the sharding, the row masks, the band / row all-reduces and the
empty-rank path are the product code; only the per-rank gridding is the CPU oracle
(TEST INFRASTRUCTURE, oracle/restate.py).  Every rank's result must equal the
single-process oracle product."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2404_17344_b200 import _native

FLAG_FROM_SPECTRUM = _native.AK_APPLY_FROM_SPECTRUM


class _OracleOp:
    """Stand-in for fastsum._Operator on one rank: C coefficient sets over the rank's
    windows, each window restricted to its masked rows.  The 'band' buffer holds the
    per-(window, RHS) band spectra (any layout works: the collectives only sum it)."""

    def __init__(self, plan, fams, R):
        from oracle import restate as Ro

        self.plan, self.fams, self.R, self.Ro = plan, fams, R, Ro
        self.shapes = [(plan.m,) * len(c) for c in plan.cols]
        self._band = torch.zeros(sum(2 * R * int(np.prod(s)) for s in self.shapes), dtype=torch.float64)

    def spectrum_only(self, V):
        Ro, p = self.Ro, self.plan
        chunks = []
        for k in range(len(p.cols)):
            for r in range(self.R):
                v = V[r].numpy()[p.rows[k]].astype(np.complex128)
                S = Ro.type1(p.nufft[k], p.geoms[k], v)
                chunks.append(torch.view_as_real(torch.from_numpy(np.ascontiguousarray(S))).reshape(-1))
        self._band.copy_(torch.cat(chunks))

    def band(self):
        return self._band

    def apply(self, V, outs, sum_windows, flags=0):
        Ro, p = self.Ro, self.plan
        if not (flags & FLAG_FROM_SPECTRUM):
            self.spectrum_only(V)
        spec = torch.view_as_complex(self._band.reshape(-1, 2)).numpy()
        off = 0
        for o in outs:
            o.zero_()
        for k, cols in enumerate(p.cols):
            q = len(cols)
            size = int(np.prod(self.shapes[k]))
            for r in range(self.R):
                S = spec[off:off + size].reshape(self.shapes[k])
                off += size
                for c, fam in enumerate(self.fams):
                    table = Ro.kernel_coefficients(fam, p.spec.ell, q, p.m)
                    vals = Ro.type2(p.nufft[k], p.geoms[k], table * S).real
                    scale = Ro.operator_scale(fam, p.spec.ell, p.spec.sigma_f)
                    outs[c][r, torch.as_tensor(p.rows[k])] += torch.from_numpy(scale * vals)


class _OraclePlan:
    def __init__(self, spec, window_set, preset, data, row_masks=None, **kw):
        from oracle import restate as Ro

        self.spec, self.m = spec, {"default": 32, "rough": 16, "fine": 64}.get(preset, preset)
        self.cols = [window_set.columns(w) for w in window_set]
        N = data.n_rows
        masks = np.ones((len(self.cols), N), bool) if row_masks is None else np.asarray(row_masks, bool)
        self.rows = [np.flatnonzero(mk) for mk in masks]
        self.nufft = [Ro.Nufft(len(c), self.m) for c in self.cols]
        self.geoms = [Ro.Geometry(self.nufft[k], data.features[self.rows[k]][:, list(c)])
                      for k, c in enumerate(self.cols)]

    def _operator(self, fams, R):
        return _OracleOp(self, fams, R)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, X, V, windows, case, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2404_17344_b200.dataset import PRESCALED, Dataset
        from paper_2404_17344_b200.distributed import CellShardedPlan, WindowShardedPlan
        from paper_2404_17344_b200.kernels import KernelSpec
        from paper_2404_17344_b200.windows import WindowSet

        ds = Dataset(X, np.zeros(X.shape[0]), tuple(f"x{i}" for i in range(X.shape[1])),
                     scaling_state=PRESCALED, d_max=3)
        ws = WindowSet(tuple(tuple(c + 1 for c in w) for w in windows), d_max=3)
        spec = KernelSpec("gauss", 0.3, 0.9)
        if case == "window":
            dp = WindowShardedPlan(spec, ws, "default", ds, plan_builder=_OraclePlan)
        else:
            G = int(case.split("_G")[1])
            dp = CellShardedPlan(spec, ws, "default", ds, window_groups=G, plan_builder=_OraclePlan)
        outs = dp.matvecs(torch.from_numpy(V), ("gauss", "der_gauss"))
        results[rank] = [o.numpy().copy() for o in outs]
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case,world", [("window", 2), ("window", 3), ("window", 4),
                                         ("cell_G1", 2), ("cell_G2", 2), ("cell_G1", 3), ("cell_G2", 4)])
def test_sharded_product_classes_match_oracle(case, world):
    """window: ranks beyond the window count (world 4 > 3 windows) own nothing and
    contribute zeros to the row all-reduce; cell_G*: G window groups x world/G cell
    slabs with the band all-reduce among a group's slabs (row-masked plans)."""
    from oracle import restate as Ro

    rng = np.random.default_rng(5)
    N = 500
    X = rng.uniform(-0.14, 0.14, size=(N, 6))
    V = rng.normal(size=(2, N))
    windows = [(0, 1, 2), (3, 4), (5,)]
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), X, V, windows, case, results), nprocs=world, join=True)
    for fam, c in (("gauss", 0), ("der_gauss", 1)):
        ref = np.stack([Ro.FastSum(fam, 0.3, 0.9, windows, X).matvec(V[r]) for r in range(2)])
        for rank in range(world):
            got = results[rank][c]
            assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref), (case, world, rank, fam)
