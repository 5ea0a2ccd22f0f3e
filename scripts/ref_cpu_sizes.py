"""The reference CPU gather (oracle/_ref) timed at several cube sizes on the
host cores (developer aid; shows its time per point falling with n)."""
import os, sys, time
sys.path.insert(0, ".")
import bench
bench._omp_env()
kind, call, label = bench.cpu_reference_runner("wave3d_r4")
sc = {"D": 0.01}
for n in [int(x) for x in sys.argv[1:]]:
    a = bench.cpu_arrays("wave3d_r4", n)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter(); call(n, sc, a); ts.append(time.perf_counter() - t0)
    print(n, ["%.3f" % t for t in ts], "GPts/s %.3f" % (n**3 / min(ts) / 1e9), flush=True)
