"""z-slab decomposition of a 3D star adjoint over ranks.

The outermost counter i is split into contiguous owned plane ranges; each rank
stores its owned planes plus R halo planes on each interior side.  The gather
form writes only owned planes, so there is no reverse accumulation; the only
exchange is the forward halo of the fields read at an i-offset (the seed u_b
and the forward state u_1; c is static and its halo is exchanged once).

Communication is torch.distributed point-to-point (NCCL on B200 over
NVLink/NVSwitch; gloo for the CPU tests): one batch_isend_irecv per step with
both neighbours.  Inputs are generated from GLOBAL indices, so every
decomposition sees the single-GPU values.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


@dataclass(frozen=True)
class Slab:
    n: int
    radius: int
    rank: int
    world: int
    own0: int  # first owned global plane
    own1: int  # one past the last owned plane
    base: int  # global plane of local plane 0 (own0 - halo below)
    nplanes: int  # local planes (owned + halos)

    @property
    def halo_lo(self) -> int:
        return self.own0 - self.base

    @property
    def halo_hi(self) -> int:
        return self.base + self.nplanes - self.own1

    @property
    def owned(self) -> int:
        return self.own1 - self.own0

    def local(self, g: int) -> int:
        return g - self.base


def decompose(n: int, radius: int, world: int, rank: int) -> Slab:
    """Contiguous, balanced split of the planes [0, n); halos of `radius`
    planes on interior sides only."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if n < world * radius:
        raise ValueError(f"n={n} too small for {world} slabs of radius {radius}")
    q, r = divmod(n, world)
    own0 = rank * q + min(rank, r)
    own1 = own0 + q + (1 if rank < r else 0)
    lo = radius if rank > 0 else 0
    hi = radius if rank < world - 1 else 0
    return Slab(n, radius, rank, world, own0, own1, own0 - lo, own1 - own0 + lo + hi)


def halo_ops(slab: Slab, fields, group=None):
    """The point-to-point ops of one halo refresh: each rank sends its R owned
    edge planes to each neighbour and receives that neighbour's into its halo.
    Planes are contiguous, so every slice is a contiguous view (no packing)."""
    R = slab.radius
    ops = []
    below, above = slab.rank - 1, slab.rank + 1
    top = slab.halo_lo + slab.owned  # local index one past the owned planes
    for f in fields:
        if below >= 0:
            ops.append(dist.P2POp(dist.isend, f[slab.halo_lo:slab.halo_lo + R], below, group))
            ops.append(dist.P2POp(dist.irecv, f[0:slab.halo_lo], below, group))
        if above < slab.world:
            ops.append(dist.P2POp(dist.isend, f[top - R:top], above, group))
            ops.append(dist.P2POp(dist.irecv, f[top:top + R], above, group))
    return ops


def exchange_halos(slab: Slab, fields, group=None) -> None:
    """Fill the halo planes of each local field (shape [nplanes, ...]) from the
    neighbours' owned edge planes: one batched isend/irecv round."""
    if slab.world == 1:
        return
    for req in dist.batch_isend_irecv(halo_ops(slab, fields, group)):
        req.wait()
