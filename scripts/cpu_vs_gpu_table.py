"""The reference CPU path timed beside the B200 kernels.

For every config family: the reference's own emitted primal / gather adjoint
/ atomic-scatter adjoint (oracle/_ref/libref_<family>.so, gcc -O2 -fopenmp;
radius 4 at -O1) on all host cores, and this repo's sm_100a kernels, at the
BASELINE size.  A CPU call that would exceed ~10 s runs on the largest cube
(square / line) that fits instead, and the row says so; rates are grid points
per second of the call.  Writes profiles/r1_cpu_vs_gpu.{json,md}.
Developer/evidence script; run on the GPU box (its host cores are the CPU).
"""
import ctypes
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_1907_02818_b200 import api  # noqa: E402
from scripts.quick_time import time_it  # noqa: E402

CASES = [("wave1d", 1 << 24, "1"), ("wave3d_c", 512, "2"), ("burgers2d", 8192, "3"),
         ("wave3d_r4", 768, "4")]
KINDS = ["primal", "adjoint", "scatter"]
CAP_S = 10.0


def host_arrays(fam, kind, n):
    d = bench.DIMS[fam]
    rng = np.random.default_rng(1)
    out = {}
    for nm in api.array_params(fam, kind):
        a = rng.standard_normal((n,) * d)
        if nm == "c":
            a = rng.uniform(1.5, 4.5, (n,) * d)
        out[nm] = a
    return out


def cpu_fn(fam, kind):
    lib = ctypes.CDLL(os.path.join(ROOT, "oracle", "_ref", f"libref_{fam}.so"))
    name = {"primal": fam, "adjoint": f"{fam}_b", "scatter": f"{fam}_scatter_b"}[kind]
    fn = getattr(lib, name)
    fn.restype = ctypes.c_int
    names = api.array_params(fam, kind)
    sc = bench.CONFIGS[dict((f, c) for f, _, c in CASES)[fam]][4]

    def call(n, arrays):
        args = [ctypes.c_int(n)] + [ctypes.c_double(sc[s]) for s in api.SCALARS[fam]] + \
               [arrays[nm].ctypes.data_as(ctypes.c_void_p) for nm in names]
        assert fn(*args) == 0
    return call


def time_cpu(fam, kind, n_full):
    d = bench.DIMS[fam]
    call = cpu_fn(fam, kind)
    n = n_full
    # probe on a quarter-size problem to estimate the full call
    n_probe = max(16, int(n_full / 2 ** (2 / d)))
    a = host_arrays(fam, kind, n_probe)
    call(n_probe, a)
    t0 = time.perf_counter()
    call(n_probe, a)
    t_probe = time.perf_counter() - t0
    est = t_probe * (n_full / n_probe) ** d
    if est > CAP_S:
        n = int(n_full * (CAP_S / est) ** (1.0 / d))
        n -= n % 4
    a = host_arrays(fam, kind, n)
    call(n, a)
    best = float("inf")
    for _ in range(2):
        t0 = time.perf_counter()
        call(n, a)
        best = min(best, time.perf_counter() - t0)
    return {"n": n, "s_per_call": best, "GPts_s": n ** d / best / 1e9}


def time_gpu(fam, kind, n, cfg):
    arrays = bench.gen_inputs(api, torch, fam, n)
    sc = bench.CONFIGS[cfg][4]
    if kind == "primal":
        dt = arrays[next(iter(arrays))].dtype
        shape = arrays[next(iter(arrays))].shape
        prim = {nm: arrays[nm] if nm in arrays else torch.randn(shape, dtype=dt, device="cuda")
                for nm in api.array_params(fam, "primal")}
        ms = time_it(lambda: api.primal(fam, n, sc, prim))
    elif kind == "adjoint":
        ms = time_it(lambda: api.adjoint(fam, n, sc, arrays))
    else:
        ms = time_it(lambda: api.scatter_adjoint(fam, n, sc, arrays), iters=5, warm=2)
    pts = n ** bench.DIMS[fam]
    return {"n": n, "ms": ms, "GPts_s": pts / ms / 1e6,
            "dtype": "f32" if fam in ("wave3d_r4", "wave3d_c") else "f64"}


def main():
    bench._omp_env()
    rows = []
    for fam, n, cfg in CASES:
        for kind in KINDS:
            g = time_gpu(fam, kind, n, cfg)
            c = time_cpu(fam, kind, n)
            rows.append({"family": fam, "kind": kind, "gpu": g, "cpu_reference": c,
                         "speedup_per_point": g["GPts_s"] / c["GPts_s"]})
            print(json.dumps(rows[-1]), flush=True)
    meta = {"cpu_model": bench.cpu_model(), "threads": int(os.environ["OMP_NUM_THREADS"]),
            "gpu": torch.cuda.get_device_name(0)}
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "cpu_vs_gpu.json"), "w") as fh:
        json.dump({"meta": meta, "rows": rows}, fh, indent=1)
    lines = [f"Reference CPU path ({meta['cpu_model']}, {meta['threads']} threads, fp64, "
             f"emitted OpenMP C) vs this repo on {meta['gpu']}.", "",
             "| family | kernel | B200 n | B200 ms | B200 GPts/s | CPU n | CPU s/call | "
             "CPU GPts/s | per-point speed-up |", "|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        g, c = r["gpu"], r["cpu_reference"]
        lines.append(f"| {r['family']} | {r['kind']} | {g['n']} ({g['dtype']}) | {g['ms']:.3f} | "
                     f"{g['GPts_s']:.1f} | {c['n']} | {c['s_per_call']:.3f} | "
                     f"{c['GPts_s']:.3f} | {r['speedup_per_point']:.0f}x |")
    with open(os.path.join(ROOT, "gpurun_out", "cpu_vs_gpu.md"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
