"""Multi-process (gloo, world_size 2, CPU) checks of the multi-GPU decompositions.

The CUDA kernels cannot run here, so each rank composes the CPU oracle with
exactly the partition functions the GPU path uses (distributed.window_partition,
distributed.row_partition) and the same collective pattern (all-reduce of the
partial products / of the per-window spread spectra); rank results must equal
the single-process product."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2404_17344_b200.distributed import row_partition, window_cost, window_partition


def test_window_partition_lpt():
    parts = window_partition([3] * 10, 8)
    assert sorted(w for p in parts for w in p) == list(range(10))
    assert max(len(p) for p in parts) == 2
    c5 = [3, 3, 3, 3, 3, 3, 2, 2, 1, 1]
    parts = window_partition(c5, 8)
    loads = [sum(window_cost(c5[w]) for w in p) for p in parts]
    assert max(loads) == window_cost(3) + window_cost(2) or max(loads) == window_cost(3)
    assert sorted(w for p in parts for w in p) == list(range(10))
    assert window_partition([3, 2], 4)[2:] == [[], []]


def test_row_partition():
    assert row_partition(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert row_partition(8, 2) == [(0, 4), (4, 8)]
    assert row_partition(1, 2) == [(0, 1), (1, 1)]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, X, v, windows, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import restate as R

    ell, sf = 0.3, 0.9
    lengths = [len(w) for w in windows]
    full = R.FastSum("gauss", ell, sf, windows, X).matvec(v)

    # window sharding: partial sums over owned windows, all-reduce
    own = window_partition(lengths, world)[rank]
    part = np.zeros_like(v)
    if own:
        part = R.FastSum("gauss", ell, sf, [windows[w] for w in own], X).matvec(v)
    t = torch.from_numpy(part.copy())
    dist.all_reduce(t)
    err_w = np.linalg.norm(t.numpy() - full) / np.linalg.norm(full)

    # point sharding: own rows spread (type-1 spectra), all-reduce, own rows interpolated
    lo, hi = row_partition(X.shape[0], world)[rank]
    fs_local = R.FastSum("gauss", ell, sf, windows, X[lo:hi])
    acc = np.zeros(hi - lo, dtype=np.complex128)
    for k, w in enumerate(windows):
        plan = fs_local.plans[len(w)]
        S = R.type1(plan, fs_local.geoms[k], v[lo:hi])
        St = torch.from_numpy(np.ascontiguousarray(S).view(np.float64).copy())
        dist.all_reduce(St)
        S_all = St.numpy().view(np.complex128).reshape(S.shape)
        acc += R.type2(plan, fs_local.geoms[k], fs_local.tables[len(w)] * S_all)
    mine = torch.from_numpy(R.operator_scale("gauss", ell, sf) * acc.real)
    sizes = [b - a for a, b in row_partition(X.shape[0], world)]
    bufs = [torch.zeros(max(sizes), dtype=torch.float64) for _ in sizes]
    pad = torch.zeros(max(sizes), dtype=torch.float64)
    pad[: mine.numel()] = mine
    dist.all_gather(bufs, pad)
    got = np.concatenate([b[:s].numpy() for b, s in zip(bufs, sizes)])
    err_p = np.linalg.norm(got - full) / np.linalg.norm(full)

    # cell sharding: per window, own whole cells (cell_partition) spread, spectra
    # all-reduced, own rows interpolated and scattered, one all-reduce of the N-vector
    from paper_2404_17344_b200.distributed import cell_partition

    part = np.zeros_like(v)
    for w in windows:
        plan = R.FastSum("gauss", ell, sf, [w], X).plans[len(w)]
        rows = cell_partition(X[:, list(w)], plan.n, world)[rank]
        fs_w = R.FastSum("gauss", ell, sf, [w], X[rows]) if len(rows) else None
        S = R.type1(plan, fs_w.geoms[0], v[rows]) if fs_w else np.zeros((plan.m,) * len(w), np.complex128)
        St = torch.from_numpy(np.ascontiguousarray(S).view(np.float64).copy())
        dist.all_reduce(St)
        if fs_w:
            S_all = St.numpy().view(np.complex128).reshape(S.shape)
            part[rows] += R.operator_scale("gauss", ell, sf) * R.type2(plan, fs_w.geoms[0],
                                                                       fs_w.tables[len(w)] * S_all).real
    t = torch.from_numpy(part)
    dist.all_reduce(t)
    err_c = np.linalg.norm(t.numpy() - full) / np.linalg.norm(full)
    q.put((rank, err_w, max(err_p, err_c)))
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_decompositions_match_single_process():
    rng = np.random.default_rng(0)
    X = rng.uniform(-0.25, 0.25, size=(301, 6)) / np.sqrt(3)
    v = rng.normal(size=301)
    windows = [(0, 1, 2), (3, 4), (5,), (1, 4, 5)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, X, v, windows, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, err_w, err_p in res:
        assert err_w <= 1e-13, (rank, err_w)
        assert err_p <= 1e-12, (rank, err_p)


def test_cell_partition_whole_cells_balanced():
    from paper_2404_17344_b200.distributed import cell_partition

    rng = np.random.default_rng(3)
    for X in (rng.uniform(-0.2, 0.2, size=(20000, 3)), rng.normal(0, 0.05, size=(5000, 2)), np.zeros((7, 1))):
        t = np.floor((X + 0.5) * 64).astype(int)
        lin = np.zeros(len(X), dtype=int)
        for a in range(X.shape[1]):
            lin = lin * 64 + t[:, a]
        for parts in (1, 2, 3, 8):
            out = cell_partition(X, 64, parts)
            assert len(out) == parts
            assert (np.sort(np.concatenate(out)) == np.arange(len(X))).all()
            owner = np.empty(len(X), dtype=int)
            for i, p in enumerate(out):
                owner[p] = i
            for c in np.unique(lin):
                assert len(set(owner[lin == c])) == 1     # no cell split across parts
    sizes = [len(p) for p in cell_partition(rng.uniform(-0.2, 0.2, size=(20000, 3)), 64, 4)]
    assert max(sizes) - min(sizes) <= 0.02 * 20000


def test_hybrid_layout():
    from paper_2404_17344_b200.distributed import hybrid_layout

    assert hybrid_layout([3] * 10, 8) == 2      # 5 + 5 windows, 4 point groups each
    assert hybrid_layout([3] * 10, 1) == 1
    assert hybrid_layout([3, 3, 3, 3], 8) == 4  # one window per group
    assert hybrid_layout([3, 3, 3], 2) == 1     # 2 + 1 is not balanced: point sharding
    assert hybrid_layout([3, 3, 3, 3, 3, 3, 2, 2, 1, 1], 8) == 2
