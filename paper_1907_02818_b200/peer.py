"""Fused halo exchange over peer memory (the fused option).

Instead of sending the R halo planes of u_1 / u_b (and c) with NCCL before
the adjoint, every rank maps its neighbours' arrays into its own address
space (CUDA IPC; NVLink peer memory between the GPUs of one box) and the
radius-4 gather kernel's own TMA loads read the input planes below / above
its owned planes straight from the neighbours (`wave3d_r4_b_slab_peer_f32`).
No separate exchange, no staging copies; the transfer rides inside the
kernel's plane pipeline.  The neighbours' planes must be final before the
call (a barrier between producing and consuming steps).

Layout: each rank's local arrays are the z-slab arrays of `slab.decompose`
(owned planes plus R halo planes on interior sides); the peer path uses only
the owned part of them, so the same arrays serve both strategies.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

from . import _lib
from .slab import Slab

FIELDS = ("c", "u_1", "u_b")


def _owned_ptr(t, sl: Slab) -> int:
    """Device address of the first owned plane of a local slab array."""
    n = sl.n
    return t.data_ptr() + (sl.own0 - sl.base) * n * n * t.element_size()


def ipc_handle(ptr: int):
    """(64-byte handle, byte offset in its allocation) of a device address."""
    h = ctypes.create_string_buffer(64)
    off = ctypes.c_longlong()
    _lib.check(_lib.lib().sgb_ipc_handle(ctypes.c_void_p(ptr), h, ctypes.byref(off)),
               "sgb_ipc_handle")
    return h.raw, off.value


def ipc_open(handle: bytes, offset: int) -> int:
    out = ctypes.c_void_p()
    _lib.check(_lib.lib().sgb_ipc_open(ctypes.create_string_buffer(handle, 64), int(offset),
                                       ctypes.byref(out)), "sgb_ipc_open")
    return out.value


@dataclass
class Neighbour:
    ptrs: dict          # field -> device address of the neighbour's first owned plane
    base: int           # global plane of that address
    nplanes: int        # owned planes the neighbour holds
    opened: list = None  # (address, offset) pairs mapped by IPC (closed by close())


@dataclass
class PeerHalo:
    sl: Slab
    lower: Neighbour | None
    upper: Neighbour | None

    def close(self):
        for nb in (self.lower, self.upper):
            if nb is not None and nb.opened:
                for ptr, off in nb.opened:
                    _lib.lib().sgb_ipc_close(ctypes.c_void_p(ptr), int(off))
                nb.opened = None


def connect(sl: Slab, arrays: dict, group=None) -> PeerHalo:
    """Collective over the ranks of a z-slab decomposition: every rank
    publishes IPC handles of the owned part of its c / u_1 / u_b arrays and
    maps its two neighbours' (torch.distributed, any backend)."""
    import torch.distributed as dist
    mine = {f: ipc_handle(_owned_ptr(arrays[f], sl)) for f in FIELDS}
    info = {"rank": sl.rank, "own0": sl.own0, "own1": sl.own1, "handles": mine}
    every = [None] * sl.world
    dist.all_gather_object(every, info, group=group)

    def open_side(r):
        if r < 0 or r >= sl.world:
            return None
        e = every[r]
        opened, ptrs = [], {}
        for f in FIELDS:
            h, off = e["handles"][f]
            p = ipc_open(h, off)
            opened.append((p, off))
            ptrs[f] = p
        return Neighbour(ptrs, e["own0"], e["own1"] - e["own0"], opened)
    return PeerHalo(sl, open_side(sl.rank - 1), open_side(sl.rank + 1))


def try_connect(sl: Slab, arrays: dict, group=None):
    """`connect` that never leaves ranks behind: every rank takes part in the
    handle exchange, then the ranks agree (MIN over a success flag) whether
    all of them could map their neighbours; returns the link or None."""
    import torch
    import torch.distributed as dist
    link, ok = None, 1
    try:
        link = connect(sl, arrays, group)
    except Exception:  # e.g. no peer access between the two GPUs
        ok = 0
    flag = torch.tensor([ok], device="cuda", dtype=torch.int32)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
    if int(flag[0]) == 0:
        if link is not None:
            link.close()
        return None
    return link


def step_sync(group=None) -> None:
    """Stream-ordered cross-rank ordering point (a 1-element NCCL all-reduce
    on the current stream): work before it on every rank precedes work after
    it on every rank, without a host synchronisation."""
    import torch
    import torch.distributed as dist
    tok = torch.zeros(1, device="cuda")
    dist.all_reduce(tok, group=group)


def emulate(slabs, arrays_per_rank):
    """Single-process stand-in for `connect` (all ranks' arrays on one device,
    neighbours addressed directly): exercises exactly the kernel path of the
    fused exchange without mutually-waiting processes."""
    out = []
    for r, sl in enumerate(slabs):
        def side(q):
            if q < 0 or q >= len(slabs):
                return None
            s2 = slabs[q]
            return Neighbour({f: _owned_ptr(arrays_per_rank[q][f], s2) for f in FIELDS},
                             s2.own0, s2.own1 - s2.own0)
        out.append(PeerHalo(sl, side(r - 1), side(r + 1)))
    return out


def adjoint(n: int, scalars: dict, arrays: dict, ph: PeerHalo, stream=None) -> None:
    """wave3d_r4 gather adjoint of the owned planes, halos read from the
    neighbours' arrays by the kernel."""
    from .api import _stream_ptr
    sl = ph.sl
    L = _lib.lib()
    own = {k: ctypes.c_void_p(_owned_ptr(arrays[k], sl))
           for k in ("c", "c_b", "u_1", "u_1_b", "u_b")}

    def nb_args(nb):
        if nb is None:
            return [None, None, None, 0, 0]
        return [ctypes.c_void_p(nb.ptrs["c"]), ctypes.c_void_p(nb.ptrs["u_1"]),
                ctypes.c_void_p(nb.ptrs["u_b"]), nb.base, nb.nplanes]
    rc = L.wave3d_r4_b_slab_peer_f32(
        int(n), float(scalars["D"]), own["c"], own["c_b"], own["u_1"], own["u_1_b"], own["u_b"],
        sl.own0, sl.own1 - sl.own0, sl.own0, sl.own1, *nb_args(ph.lower), *nb_args(ph.upper),
        _stream_ptr(stream))
    _lib.check(rc, "wave3d_r4_b_slab_peer_f32")
