"""Sustained-run probe (developer aid): per-step time of the cfg 4 gather
adjoint over a long back-to-back run, with the SM clock, board power and
throttle reasons sampled alongside, and the same for a plain device copy of
the same byte volume -- separates clock / power effects from the kernel."""
import statistics
import sys
import threading
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1907_02818_b200 import api  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 600
n = 768
cfg = bench.CONFIGS["4"]
arrays = bench.gen_inputs(api, torch, "wave3d_r4", n)
torch.cuda.synchronize()

import pynvml  # noqa: E402
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
samples = []
stop = threading.Event()


def sampler():
    while not stop.is_set():
        t = time.perf_counter()
        try:
            clk = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
            mclk = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM)
            pw = pynvml.nvmlDeviceGetPowerUsage(h) / 1e3
            r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
            samples.append((t, clk, mclk, pw, r))
        except Exception:
            pass
        time.sleep(0.005)


def run(label, fn, steps, sync_each=False):
    samples.clear()
    stop.clear()
    th = threading.Thread(target=sampler, daemon=True)
    th.start()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    t0 = time.perf_counter()
    evs[0].record()
    for i in range(steps):
        fn()
        evs[i + 1].record()
        if sync_each:
            evs[i + 1].synchronize()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    stop.set()
    th.join()
    ms = [evs[i].elapsed_time(evs[i + 1]) for i in range(steps)]
    print(f"== {label}: {steps} steps, total {sum(ms):.1f} ms, wall {1e3 * (t1 - t0):.1f} ms")
    blk = max(1, steps // 10)
    acc = 0.0
    for b in range(0, steps, blk):
        seg = ms[b:b + blk]
        ta, tb = t0 + acc / 1e3, t0 + (acc + sum(seg)) / 1e3
        acc += sum(seg)
        ss = [s for s in samples if ta <= s[0] < tb]
        clk = statistics.median([s[1] for s in ss]) if ss else None
        mclk = statistics.median([s[2] for s in ss]) if ss else None
        pw = statistics.median([s[3] for s in ss]) if ss else None
        rs = sorted({s[4] for s in ss})
        print(f"  steps {b:4d}-{b + len(seg) - 1:4d}: {statistics.median(seg):.3f} ms/step "
              f"sm {clk} MHz mem {mclk} MHz power {pw} W reasons {[hex(x) for x in rs]}")


sc = cfg[4]
run("adjoint back-to-back", lambda: api.adjoint("wave3d_r4", n, sc, arrays), steps)
time.sleep(2)
run("adjoint sync each step", lambda: api.adjoint("wave3d_r4", n, sc, arrays), steps // 3,
    sync_each=True)
time.sleep(2)
# copy with the same DRAM volume as one gather step (12.7 GB): 6.34 GB read + written
a = torch.empty(int(6.34e9 / 4 / 2), dtype=torch.float32, device="cuda")
b = torch.empty_like(a)
run("copy 12.7 GB back-to-back", lambda: (b.copy_(a), a.copy_(b)), steps)
