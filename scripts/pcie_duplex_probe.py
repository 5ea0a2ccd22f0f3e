"""PCIe copy rates of this box: H2D alone, D2H alone, and both at once (the
host-state sweep's pattern: 2 bytes in per byte out), pinned host memory.
python scripts/pcie_duplex_probe.py [GiB]"""
import sys

import torch

gib = float(sys.argv[1]) if len(sys.argv) > 1 else 4.0
n = int(gib * 2**30 / 4)
h_in = [torch.empty(n, dtype=torch.float32).pin_memory() for _ in range(2)]
h_out = torch.empty(n, dtype=torch.float32).pin_memory()
d_in = [torch.empty(n, dtype=torch.float32, device="cuda") for _ in range(2)]
d_out = torch.empty(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
CH = 64


def run(h2d, d2h):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    s1.wait_stream(torch.cuda.current_stream())
    s2.wait_stream(torch.cuda.current_stream())
    step = n // CH
    for c in range(CH):
        sl = slice(c * step, (c + 1) * step)
        if h2d:
            with torch.cuda.stream(s1):
                for k in range(2):
                    d_in[k][sl].copy_(h_in[k][sl], non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2):
                h_out[sl].copy_(d_out[sl], non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / 1e3


for name, h2d, d2h in (("H2D alone", 1, 0), ("D2H alone", 0, 1), ("both", 1, 1)):
    run(h2d, d2h)
    t = min(run(h2d, d2h) for _ in range(3))
    gb_in, gb_out = 2 * n * 4 / 1e9 * h2d, n * 4 / 1e9 * d2h
    print(f"{name:10s} {t * 1e3:8.1f} ms  H2D {gb_in / t:5.1f} GB/s  D2H {gb_out / t:5.1f} GB/s",
          flush=True)
