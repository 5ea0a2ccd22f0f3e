"""Multi-rank z-slab host logic on CPU (gloo, world_size 2 and 3).

Checks the decomposition arithmetic and that one halo refresh leaves every
rank's local planes (owned + halos) equal to the corresponding planes of the
global field -- the precondition under which the slab kernels reproduce the
single-GPU result bit for bit (tests/test_gpu_parity.py::test_slabs_*).
"""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1907_02818_b200 import slab as slabmod


def test_decompose_partitions_planes():
    for n in (17, 64, 768, 1024):
        for world in (1, 2, 3, 4, 8):
            if n < world * 4:
                continue
            slabs = [slabmod.decompose(n, 4, world, r) for r in range(world)]
            assert slabs[0].own0 == 0 and slabs[-1].own1 == n
            for a, b in zip(slabs, slabs[1:]):
                assert a.own1 == b.own0
            sizes = [s.owned for s in slabs]
            assert max(sizes) - min(sizes) <= 1
            for s in slabs:
                assert s.halo_lo == (4 if s.rank > 0 else 0)
                assert s.halo_hi == (4 if s.rank < world - 1 else 0)
                assert s.base + s.nplanes <= n and s.base >= 0


def _free_port():
    with socket.socket() as sck:
        sck.bind(("127.0.0.1", 0))
        return sck.getsockname()[1]


def _worker(rank, world, port, n, radius, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = torch.arange(n * 6 * 5, dtype=torch.float32).reshape(n, 6, 5)
        g2 = -g
        sl = slabmod.decompose(n, radius, world, rank)
        loc = torch.full((sl.nplanes, 6, 5), float("nan"))
        loc2 = torch.full((sl.nplanes, 6, 5), float("nan"))
        own = slice(sl.halo_lo, sl.halo_lo + sl.owned)
        loc[own] = g[sl.own0:sl.own1]
        loc2[own] = g2[sl.own0:sl.own1]
        slabmod.exchange_halos(sl, [loc, loc2])
        ok = torch.equal(loc, g[sl.base:sl.base + sl.nplanes]) and \
            torch.equal(loc2, g2[sl.base:sl.base + sl.nplanes])
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,radius", [(2, 20, 4), (3, 17, 4), (2, 9, 1)])
def test_halo_exchange_gloo(world, n, radius):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, radius, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(res.values()), res


def _prefetch_worker(rank, world, port, n, radius, steps, q):
    """drivers.HaloPrefetch's schedule with the real exchange (gloo, CPU
    tensors): each step's compute must see its own step's owned planes and the
    neighbours' edge planes of the SAME step in its halos, from the set the
    double buffering assigns it -- the data routing of the pipelined exchange
    in a true multi-process run (the CUDA stream / event ordering on top of it
    is covered on the B200, tests/test_drivers_gpu.py)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1907_02818_b200 import drivers
        sl = slabmod.decompose(n, radius, world, rank)
        shape = (sl.nplanes, 6, 5)

        def glob(t, field):  # the step-t global field, planes [base, base + nplanes)
            g = torch.arange(n * 6 * 5, dtype=torch.float64).reshape(n, 6, 5)
            return g + 1e6 * t + (0.5 if field == "u_b" else 0.0)

        def regen(fs, t):  # owned planes only; halo planes poisoned
            for f, tens in fs.items():
                tens.fill_(float("nan"))
                tens[sl.halo_lo:sl.halo_lo + sl.owned] = glob(t, f)[sl.own0:sl.own1]

        seen = []

        def compute(inputs, t):
            ok = all(torch.equal(inputs[f], glob(t, f)[sl.base:sl.base + sl.nplanes])
                     for f in ("u_1", "u_b"))
            seen.append(ok)

        arrays = {f: torch.zeros(shape, dtype=torch.float64) for f in ("c", "u_1", "u_b")}
        pf = drivers.HaloPrefetch("wave3d_r4", n, {"D": 0.01}, arrays, sl, regen=regen,
                                  compute=compute)
        for _ in range(steps):
            pf.step()
        pf.close()
        q.put((rank, len(seen) == steps and all(seen)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,radius", [(2, 20, 4), (3, 17, 4)])
def test_halo_prefetch_schedule_gloo(world, n, radius):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_prefetch_worker, args=(r, world, port, n, radius, 5, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(res.values()), res
