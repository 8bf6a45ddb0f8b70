"""GPU: the multi-GPU decompositions (distributed.py) with two ranks on the one
available device, exchanging through gloo (host-side collectives; the ranks'
kernels never wait on each other), and with one rank over NCCL (the production
backend: communicator set-up, subgroups and device all-reduces on the B200).  Checks the real sharded code paths --
SPECTRUM_ONLY spread + band all-reduce + FROM_SPECTRUM interpolation (point
sharding) and the LPT window split + all-reduce (window sharding) -- against the
single-process product; with 4 ranks also the 2 x 2 hybrid (window groups x
point groups); and the cell-slab layout (CellShardedPlan) for every group count."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, X, V, q, backend="gloo"):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", 0))
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2404_17344_b200.dataset import PRESCALED, Dataset
        from paper_2404_17344_b200.distributed import (CellShardedPlan, HybridShardedPlan, PointShardedPlan,
                                                       WindowShardedPlan)
        from paper_2404_17344_b200.fastsum import build_plan, fast_matvecs
        from paper_2404_17344_b200.kernels import KernelSpec
        from paper_2404_17344_b200.windows import WindowSet

        ds = Dataset(X, np.zeros(X.shape[0]), tuple(f"x{i}" for i in range(X.shape[1])), scaling_state=PRESCALED,
                     d_max=3)
        ws = WindowSet(((1, 2, 3), (4, 5, 6), (2, 5), (7,)), d_max=3)
        spec = KernelSpec("gauss", 0.3, 0.9)
        ref = fast_matvecs(build_plan(spec, ws, "default", ds), V, dell=True)
        Vd = torch.as_tensor(V, device="cuda")
        errs = {}
        for exchange in ("band", "grid"):
            pp = PointShardedPlan(spec, ws, "default", ds, exchange=exchange)
            k_rows = pp.matvec(Vd[0]).cpu().numpy()
            errs[f"point_{exchange}_K"] = np.linalg.norm(k_rows - ref["K"][0]) / np.linalg.norm(ref["K"][0])
            local = pp.matvecs_local(Vd[:, pp.lo:pp.hi].contiguous(), ("gauss", "der_gauss"))
            for name, o in zip(("K", "dK_dell"), local):
                r = ref[name][:, pp.lo:pp.hi]
                errs[f"point_{exchange}_local_{name}"] = np.linalg.norm(o.cpu().numpy() - r) / np.linalg.norm(r)
        if world <= 2:
            wp = WindowShardedPlan(spec, ws, "default", ds)
            outs = wp.matvecs(Vd, ("gauss", "der_gauss"))
            for name, o in zip(("K", "dK_dell"), outs):
                errs[f"window_{name}"] = np.linalg.norm(o.cpu().numpy() - ref[name]) / np.linalg.norm(ref[name])
        for G in sorted(g for g in {1, 2, world} if world % g == 0):
            hp = HybridShardedPlan(spec, ws, "default", ds, window_groups=G)
            k_rows = hp.matvec(Vd[0]).cpu().numpy()
            errs[f"hybrid{G}_K"] = np.linalg.norm(k_rows - ref["K"][0]) / np.linalg.norm(ref["K"][0])
            local = hp.matvecs_local(Vd[:, hp.lo:hp.hi].contiguous(), ("gauss", "der_gauss"))
            for name, o in zip(("K", "dK_dell"), local):
                r = ref[name][:, hp.lo:hp.hi]
                errs[f"hybrid{G}_local_{name}"] = np.linalg.norm(o.cpu().numpy() - r) / np.linalg.norm(r)
        for G in sorted(g for g in {1, 2, world} if world % g == 0):
            cp = CellShardedPlan(spec, ws, "default", ds, window_groups=G)
            outs = cp.matvecs(Vd, ("gauss", "der_gauss"))
            for name, o in zip(("K", "dK_dell"), outs):
                errs[f"cell{G}_{name}"] = np.linalg.norm(o.cpu().numpy() - ref[name]) / np.linalg.norm(ref[name])
            k1 = cp.matvec(Vd[1]).cpu().numpy()
            errs[f"cell{G}_matvec"] = np.linalg.norm(k1 - ref["K"][1]) / np.linalg.norm(ref["K"][1])
        q.put((rank, errs))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,backend", [(2, "gloo"), (4, "gloo"), (1, "nccl")])
def test_ranks_on_one_device_match_single_process(cuda, world, backend):
    import torch.multiprocessing as mp

    rng = np.random.default_rng(21)
    X = rng.uniform(-0.14, 0.14, size=(5001, 7))   # odd N: unequal row blocks
    V = rng.normal(size=(3, 5001))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, X, V, q, backend)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, errs in results:
        for key, err in errs.items():
            assert err <= 1e-12, (rank, key, err)
