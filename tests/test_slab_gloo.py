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
