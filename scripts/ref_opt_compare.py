"""Reference radius-4 CPU adjoint: the -O1 and -O2 builds of the emitted code
timed on this host (developer aid):  python scripts/ref_opt_compare.py [n]"""
import ctypes
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 768
bench._omp_env()
a = bench.cpu_arrays("wave3d_r4", n)
names = ["c", "c_b", "u_1", "u_1_b", "u_b"]
for lib in ("libref_wave3d_r4.so", "libref_wave3d_r4_O2.so"):
    p = os.path.join("oracle", "_ref", lib)
    if not os.path.exists(p):
        print(lib, "missing")
        continue
    fn = ctypes.CDLL(p).wave3d_r4_b
    args = [ctypes.c_int(n), ctypes.c_double(0.01)] + \
           [a[k].ctypes.data_as(ctypes.c_void_p) for k in names]
    fn(*args)
    best = 1e9
    for _ in range(3):
        t0 = time.perf_counter()
        fn(*args)
        best = min(best, time.perf_counter() - t0)
    print(f"{lib}: {best:.3f} s per call, {n ** 3 / best / 1e9:.3f} GPts/s "
          f"({os.environ['OMP_NUM_THREADS']} threads)", flush=True)
