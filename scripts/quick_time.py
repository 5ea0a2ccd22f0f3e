"""Scratch timing of the gather-adjoint kernels (developer aid, not the bench)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1907_02818_b200 import api  # noqa: E402


def time_it(fn, iters=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(iters):
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    cases = [("wave3d_r4", 768, torch.float32, 28), ("wave3d_c", 512, torch.float32, 36),
             ("wave1d", 1 << 24, torch.float64, 72), ("burgers2d", 8192, torch.float64, 32),
             ("wave3d_r4", 1024, torch.float32, 28)]
    only = sys.argv[1:]
    for name, n, dt, bpp in cases:
        if only and f"{name}:{n}" not in only:
            continue
        d = api.FAMILIES[name]
        shape = (n,) * d
        arrays = {}
        for i, nm in enumerate(api.array_params(name, "adjoint")):
            t = torch.empty(shape, dtype=dt, device="cuda")
            api.fill_random(t, 0, 1, i, "normal", 0.0, 1.0)
            arrays[nm] = t
        if "c" in arrays:
            api.fill_random(arrays["c"], 0, 1, 99, "uniform", 1.5, 3.0)
        sc = {"D": 0.01 if name == "wave3d_r4" else 0.1, "C": 0.2}
        for kind in ("adjoint", "scatter"):
            if kind == "scatter" and (n > 800 or only):
                continue
            fn = (lambda: api.adjoint(name, n, sc, arrays)) if kind == "adjoint" else \
                (lambda: api.scatter_adjoint(name, n, sc, arrays))
            ms = time_it(fn, iters=(10 if kind == "scatter" else 20) if not only else 3, warm=3 if not only else 1)
            pts = n ** d
            print(f"{name:10s} n={n:9d} {kind:8s} {ms:8.3f} ms  {pts / ms / 1e6:8.2f} GPts/s  "
                  f"{pts * bpp / ms / 1e6:8.1f} GB/s", flush=True)
        del arrays
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
