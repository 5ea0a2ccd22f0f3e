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


# ---------------------------------------------------------------------------
# The library's own z-slab plan (sgb_slab_*, include/stencilgrad_b200.h): the
# exchange lives in the C ABI (NCCL or the CUDA-IPC copy-engine transport) and
# this class is a thin caller.  torch.distributed (any backend) is only the
# out-of-band channel for the NCCL unique id / the IPC blobs.
TRANSPORTS = {"nccl": 1, "ipc": 2}
STEP_FRESH, STEP_OVERLAP, STEP_NO_EXCHANGE = 1, 2, 4
FIELD_MASK = {"c": 1, "u_1": 2, "u_b": 4}


def c_decompose(n: int, radius: int, world: int, rank: int) -> Slab:
    """sgb_slab_decompose (the C plan's geometry) as a Slab."""
    import ctypes
    from . import _lib
    o0, o1, b, npl = (ctypes.c_int() for _ in range(4))
    _lib.check(_lib.lib().sgb_slab_decompose(n, radius, world, rank, ctypes.byref(o0),
                                             ctypes.byref(o1), ctypes.byref(b),
                                             ctypes.byref(npl)), "sgb_slab_decompose")
    return Slab(n, radius, rank, world, o0.value, o1.value, b.value, npl.value)


class SlabPlan:
    """One rank's sgb_slab plan.  `arrays` (set 0) and `arrays1` (optional
    second input set: u_1 / u_b for a pipelined driver) are this rank's local
    slab tensors ([nplanes, n, n]); they are bound once and must outlive the
    plan.  connect() is collective over the default (or given) process group."""

    def __init__(self, family: str, n: int, arrays: dict, rank: int, world: int,
                 transport: str = "ipc", arrays1: dict | None = None, group=None):
        import ctypes
        import torch
        from . import _lib
        self._lib, self._ct = _lib, ctypes
        dt = next(iter(arrays.values())).dtype
        self.dtype_bytes = 8 if dt == torch.float64 else 4
        self.family, self.n, self.rank, self.world = family, n, rank, world
        self.transport = transport
        uid = None
        if transport == "nccl":
            import torch.distributed as dist
            buf = ctypes.create_string_buffer(128)
            if rank == 0:
                _lib.check(_lib.lib().sgb_nccl_unique_id(buf), "sgb_nccl_unique_id")
            obj = [buf.raw if rank == 0 else None]
            if world > 1:
                dist.broadcast_object_list(obj, src=0, group=group)
            uid = ctypes.create_string_buffer(obj[0], 128)
        self._p = _lib.lib().sgb_slab_create(family.encode(), n, self.dtype_bytes, rank, world,
                                             TRANSPORTS[transport], uid)
        if not self._p:
            raise _lib.StencilError(_lib.lib().sgb_last_error().decode())
        b, npl, o0, o1 = (ctypes.c_int() for _ in range(4))
        _lib.lib().sgb_slab_geometry(ctypes.c_void_p(self._p), ctypes.byref(b), ctypes.byref(npl),
                                     ctypes.byref(o0), ctypes.byref(o1))
        R = 4 if family == "wave3d_r4" else 1
        self.slab = Slab(n, R, rank, world, o0.value, o1.value, b.value, npl.value)
        self.keep = [arrays, arrays1]
        for s, arrs in enumerate((arrays, arrays1)):
            for nm, t in (arrs or {}).items():
                if tuple(t.shape) != (self.slab.nplanes, n, n) or not t.is_contiguous():
                    raise _lib.StencilError(f"SlabPlan: '{nm}' must be a contiguous "
                                            f"[{self.slab.nplanes}, {n}, {n}] tensor")
                _lib.check(_lib.lib().sgb_slab_bind(ctypes.c_void_p(self._p), s, nm.encode(),
                                                    ctypes.c_void_p(t.data_ptr())),
                           "sgb_slab_bind")
        self.group = group

    def connect(self):
        """IPC: publish this rank's blob, map the neighbours' (collective)."""
        if self.transport != "ipc" or self.world == 1:
            return self
        import torch.distributed as dist
        ct, L = self._ct, self._lib.lib()
        nbytes = ct.c_longlong(0)
        self._lib.check(L.sgb_slab_ipc_export(ct.c_void_p(self._p), None, ct.byref(nbytes)),
                        "sgb_slab_ipc_export")
        blob = ct.create_string_buffer(nbytes.value)
        self._lib.check(L.sgb_slab_ipc_export(ct.c_void_p(self._p), blob, ct.byref(nbytes)),
                        "sgb_slab_ipc_export")
        every = [None] * self.world
        dist.all_gather_object(every, blob.raw, group=self.group)
        lo = ct.create_string_buffer(every[self.rank - 1]) if self.rank > 0 else None
        hi = ct.create_string_buffer(every[self.rank + 1]) if self.rank < self.world - 1 else None
        self._lib.check(L.sgb_slab_ipc_connect(ct.c_void_p(self._p), lo, hi),
                        "sgb_slab_ipc_connect")
        # probe both peer paths (remote stream-memop write, peer copy) before
        # any step can wait on them: a box without a usable peer path fails
        # here instead of hanging in the first exchange
        dist.barrier(group=self.group)
        rc0 = L.sgb_slab_ipc_probe(ct.c_void_p(self._p), 0)
        dist.barrier(group=self.group)
        rc1 = L.sgb_slab_ipc_probe(ct.c_void_p(self._p), 1) if rc0 == 0 else rc0
        msg = L.sgb_last_error().decode(errors="replace") if rc1 else ""
        verdicts = [None] * self.world
        dist.all_gather_object(verdicts, (rc1, msg), group=self.group)
        bad = [(r, v) for r, v in enumerate(verdicts) if v[0] != 0]
        if bad:  # every rank refuses the transport together
            r, (rc, m) = bad[0]
            raise self._lib.StencilError(f"sgb_slab_ipc_probe failed on rank {r} ({rc}): {m}")
        return self

    def release(self):
        """IPC watchdog: drain an exchange that never completed (the plan's
        results are void afterwards; close it)."""
        if self.transport == "ipc" and getattr(self, "_p", None):
            self._lib.check(self._lib.lib().sgb_slab_release(self._ct.c_void_p(self._p)),
                            "sgb_slab_release")

    def _stream(self, stream):
        import torch
        s = stream if stream is not None else torch.cuda.current_stream()
        return self._ct.c_void_p(s.cuda_stream)

    def halo_start(self, fields=("u_1", "u_b"), set_=0, stream=None):
        mask = 0
        for f in fields:
            mask |= FIELD_MASK[f]
        self._lib.check(self._lib.lib().sgb_slab_halo_start(self._ct.c_void_p(self._p), set_, mask,
                                                            self._stream(stream)),
                        "sgb_slab_halo_start")

    def halo_wait(self, set_=0, stream=None):
        self._lib.check(self._lib.lib().sgb_slab_halo_wait(self._ct.c_void_p(self._p), set_,
                                                           self._stream(stream)),
                        "sgb_slab_halo_wait")

    def step(self, scalars: dict, set_=0, fresh=False, overlap=False, exchanged=False,
             stream=None):
        """One reverse step over the owned planes (exchange of u_1 / u_b, then
        the gather; `exchanged`: the halos of `set_` were refreshed by an
        earlier halo_start -- wait for it, then one launch)."""
        from . import api
        flags = (STEP_FRESH if fresh else 0) | (STEP_OVERLAP if overlap else 0) | \
            (STEP_NO_EXCHANGE if exchanged else 0)
        sc = (self._ct.c_double * 2)(*[float(scalars[s]) for s in api.SCALARS[self.family]])
        self._lib.check(self._lib.lib().sgb_slab_step(self._ct.c_void_p(self._p), set_, sc, flags,
                                                      self._stream(stream)), "sgb_slab_step")

    def close(self):
        if getattr(self, "_p", None):
            import torch
            torch.cuda.synchronize()
            self._lib.lib().sgb_slab_destroy(self._ct.c_void_p(self._p))
            self._p = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
