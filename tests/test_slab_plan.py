"""The library's multi-GPU z-slab plan (sgb_slab_*; VERDICT r1 'move
multi-GPU into the library'): geometry equals slab.decompose; the C++ caller
(tests/cpp/test_slab_ipc.cpp) runs W ranks as W processes on the one GPU with
the CUDA-IPC copy-engine transport -- halos NaN-poisoned, refreshed only by
the plan's exchange -- in three schedules and matches the single-GPU result
bitwise; the Python caller (slab.SlabPlan) the same over gloo-exchanged blobs;
the NCCL transport initialises a 1-rank communicator (ranks sharing one GPU
cannot form an NCCL communicator, so its exchange runs on the 8-GPU box)."""
import itertools
import os
import socket
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1907_02818_b200")


def test_c_geometry_equals_decompose():
    from paper_1907_02818_b200 import slab
    for n, R, W in itertools.product([16, 37, 72, 768, 1024], [1, 4], [1, 2, 3, 4, 8]):
        if n < W * R:
            continue
        for r in range(W):
            assert slab.c_decompose(n, R, W, r) == slab.decompose(n, R, W, r)


def _build_cpp(out):
    from paper_1907_02818_b200 import build as b
    b.build()
    cmd = ["g++", "-std=c++17", "-O2", os.path.join(ROOT, "tests", "cpp", "test_slab_ipc.cpp"),
           "-I" + os.path.join(ROOT, "include"), "-I/usr/local/cuda/include", "-L" + LIBDIR,
           "-lstencilgrad_b200", "-L/usr/local/cuda/lib64", "-lcudart",
           "-Wl,-rpath," + LIBDIR, "-Wl,-rpath,/usr/local/cuda/lib64", "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


def test_cpp_slab_caller_builds(tmp_path):
    assert os.path.exists(_build_cpp(str(tmp_path / "test_slab_ipc")))


@pytest.mark.gpu
@pytest.mark.parametrize("world,n,steps", [(2, 72, 4), (3, 108, 3), (4, 96, 3)])
def test_cpp_slab_ipc_processes_one_gpu(tmp_path, world, n, steps):
    exe = _build_cpp(str(tmp_path / "test_slab_ipc"))
    r = subprocess.run([exe, str(world), str(n), str(steps)], capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert f"world {world}" in r.stdout and "ok" in r.stdout.splitlines()[-1]


@pytest.mark.gpu
@pytest.mark.parametrize("transport", ["nccl", "ipc"])
def test_one_rank_plan_equals_single_gpu(transport):
    """world = 1: the plan's step is the single-GPU fresh gather (NCCL: a
    1-rank communicator from a real unique id)."""
    import torch
    import torch.distributed as dist
    from paper_1907_02818_b200 import api, drivers, slab
    n = 64
    a = drivers.alloc("wave3d_r4", n)
    drivers.init_static("wave3d_r4", a, n, 0)
    drivers.regen_state(a["u_1"], n, 0, 0, 4)
    drivers.regen_seed(a["u_b"], n, 0, 0)
    b = {k: v.clone() for k, v in a.items()}
    if transport == "nccl" and not dist.is_initialized():
        pass  # world 1: no broadcast needed
    plan = slab.SlabPlan("wave3d_r4", n, a, 0, 1, transport).connect()
    plan.step({"D": 0.01}, fresh=True)
    api.adjoint_fresh("wave3d_r4", n, {"D": 0.01}, b)
    torch.cuda.synchronize()
    plan.close()
    for k in ("c_b", "u_1_b"):
        assert torch.equal(a[k], b[k]), k


def _py_rank(rank, world, port, n, steps, q):
    try:
        import torch
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        from paper_1907_02818_b200 import api, drivers, slab
        fam, D = "wave3d_r4", 0.01
        ref = drivers.run_independent(n, steps, seed=0, D=D)
        want = {k: ref[k].clone() for k in ("c_b", "u_1_b")}
        del ref
        sl = slab.c_decompose(n, 4, world, rank)
        loc = drivers.alloc(fam, n, sl)
        loc1 = {k: torch.full_like(loc[k], float("nan")) for k in ("u_1", "u_b")}
        for k in ("c", "u_1", "u_b"):
            loc[k].fill_(float("nan"))
        drivers.init_static(fam, loc, n, 0, sl)  # c on every local plane...
        loc["c"][:sl.halo_lo] = float("nan")     # ...halos must come from the exchange
        loc["c"][sl.own1 - sl.base:] = float("nan")
        plan = slab.SlabPlan(fam, n, loc, rank, world, "ipc", arrays1=loc1).connect()
        plan.halo_start(("c",))
        own = slice(sl.own0 - sl.base, sl.own1 - sl.base)
        sets = [loc, {**loc, **loc1}]

        owned = slab.Slab(n, 4, rank, world, sl.own0, sl.own1, sl.own0, sl.owned)

        def regen(t, set_):  # step t's inputs on the OWNED planes of set_
            s = sets[set_]
            drivers.regen_state(s["u_1"][own], n, t, 0, 4, owned)
            drivers.regen_seed(s["u_b"][own], n, t, 0, owned)
        ok = True
        for mode in ("serial", "overlap", "pipelined"):
            loc["c_b"].zero_()
            if mode != "pipelined":
                for t in range(steps):
                    regen(t, 0)
                    plan.step({"D": D}, fresh=True, overlap=mode == "overlap")
            else:
                regen(0, 0)
                plan.halo_start(set_=0)
                for t in range(steps):
                    if t + 1 < steps:
                        regen(t + 1, (t + 1) % 2)
                        plan.halo_start(set_=(t + 1) % 2)
                    plan.step({"D": D}, set_=t % 2, fresh=True, exchanged=True)
            torch.cuda.synchronize()
            for k in ("c_b", "u_1_b"):
                ok &= torch.equal(loc[k][own], want[k][sl.own0:sl.own1])
        dist.barrier()
        if rank == 0:
            # the bench watchdog's path: an exchange whose neighbour never
            # joins stays queued; releasing this rank's flags drains it
            import time
            plan.halo_start(set_=1)
            plan.halo_wait(set_=1)
            ev = torch.cuda.Event()
            ev.record()
            time.sleep(1.0)
            stuck = not ev.query()
            plan.release()
            t0 = time.time()
            while not ev.query() and time.time() - t0 < 30:
                time.sleep(0.01)
            ok &= stuck and ev.query()
        dist.barrier()
        plan.close()
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, bool(ok), ""))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, False, traceback.format_exc()[-1500:]))


@pytest.mark.gpu
@pytest.mark.parametrize("world,n,steps", [(2, 72, 3), (3, 96, 2)])
def test_python_slab_plan_ipc_processes_one_gpu(world, n, steps):
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_py_rank, args=(r, world, port, n, steps, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
