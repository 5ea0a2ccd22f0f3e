"""Fused halo exchange over peer memory (paper_1907_02818_b200/peer.py).

(1) Single-process emulation of N ranks on one GPU (the profiling guide's
    recommended stand-in: one process, every rank's arrays addressed
    directly): each rank's radius-4 gather reads its halo planes straight
    from the neighbours' arrays; its own halo planes are poisoned with NaN to
    prove they are never read; owned planes equal the single-GPU result bit
    for bit.
(2) The IPC plumbing with two processes on the one GPU (gloo for the handle
    exchange; no kernel waits on another process): each rank maps its
    neighbour's arrays with cudaIpcOpenMemHandle and checks its owned planes
    against the full-grid adjoint it computes itself.
"""
import os
import socket

import pytest

pytestmark = pytest.mark.gpu


def _global_inputs(torch, api, n, seed=3):
    a = {nm: torch.empty((n, n, n), device="cuda")
         for nm in api.array_params("wave3d_r4", "adjoint")}
    api.fill_layered(a["c"], n, 8, 1.5, 4.5, seed)
    api.fill_normal3d(a["u_1"], n, 4, seed, 1)
    api.fill_normal3d(a["u_b"], n, 0, seed, 3)
    api.fill_normal3d(a["c_b"], n, 0, seed, 5)
    api.fill_normal3d(a["u_1_b"], n, 0, seed, 6)
    return a


@pytest.mark.parametrize("n,world", [(68, 2), (136, 3), (96, 4), (64, 2)])
def test_peer_halo_emulated_ranks_bitwise(n, world):
    import torch
    from paper_1907_02818_b200 import api, peer, slab
    full = _global_inputs(torch, api, n)
    ref = {k: v.clone() for k, v in full.items()}
    api.adjoint("wave3d_r4", n, {"D": 0.01}, ref)
    slabs = [slab.decompose(n, 4, world, r) for r in range(world)]
    local = []
    for sl in slabs:
        loc = {k: v[sl.base:sl.base + sl.nplanes].clone() for k, v in full.items()}
        for k in ("c", "u_1", "u_b"):  # halo planes: never read by the peer path
            loc[k][:sl.halo_lo] = float("nan")
            loc[k][sl.own1 - sl.base:] = float("nan")
        local.append(loc)
    links = peer.emulate(slabs, local)
    for r, sl in enumerate(slabs):
        peer.adjoint(n, {"D": 0.01}, local[r], links[r])
    torch.cuda.synchronize()
    for r, sl in enumerate(slabs):
        a, b = sl.own0 - sl.base, sl.own1 - sl.base
        for k in ("c_b", "u_1_b"):
            assert torch.equal(local[r][k][a:b], ref[k][sl.own0:sl.own1]), (r, k)


def _ipc_rank(rank, world, port, n, q):
    try:
        import torch
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        from paper_1907_02818_b200 import api, peer, slab
        full = _global_inputs(torch, api, n)
        ref = {k: v.clone() for k, v in full.items()}
        api.adjoint("wave3d_r4", n, {"D": 0.01}, ref)
        sl = slab.decompose(n, 4, world, rank)
        loc = {k: v[sl.base:sl.base + sl.nplanes].clone() for k, v in full.items()}
        del full
        torch.cuda.synchronize()
        link = peer.connect(sl, loc)
        dist.barrier()  # every rank's planes are final before anyone reads them
        peer.adjoint(n, {"D": 0.01}, loc, link)
        torch.cuda.synchronize()
        dist.barrier()  # nobody frees arrays a neighbour may still be reading
        a, b = sl.own0 - sl.base, sl.own1 - sl.base
        ok = all(torch.equal(loc[k][a:b], ref[k][sl.own0:sl.own1]) for k in ("c_b", "u_1_b"))
        link.close()
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, ok, ""))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, False, repr(e)))


def test_peer_halo_ipc_two_processes_one_gpu():
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_rank, args=(r, 2, port, 72, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
