"""cfg 5 step, serial vs pipelined on one GPU (developer aid): the serial step
regenerates u_1 / u_b and then runs the fresh gather; the pipelined form keeps
two u_1 / u_b sets and regenerates step t+1's set on a low-priority side
stream while step t's gather (high priority) reads the other set -- the same
double buffering drivers.HaloPrefetch does at N > 1.  The v8 interior CTA
leaves room for one generator block per SM, so the generator soaks up the
DRAM and issue slots the gather leaves idle.
python scripts/cfg5_pipe_time.py [n] [steps] [rounds]"""
import statistics
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1907_02818_b200 import api, drivers  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 5
fam, sc, R = "wave3d_r4", {"D": 0.01}, 4
a = drivers.alloc(fam, n)
drivers.init_static(fam, a, n, 0)
sets = [{"u_1": a["u_1"], "u_b": a["u_b"]},
        {"u_1": torch.empty_like(a["u_1"]), "u_b": torch.empty_like(a["u_b"])}]
lo_pri, hi_pri = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") else (0, -1)
main = torch.cuda.Stream(priority=-1)
side = torch.cuda.Stream(priority=0)


def serial(k):
    with torch.cuda.stream(main):
        for t in range(k):
            drivers.regen_step(a["u_1"], a["u_b"], n, t, 0, R)
            api.adjoint_fresh(fam, n, sc, a)


def pipelined(k):
    with torch.cuda.stream(main):
        drivers.regen_step(sets[0]["u_1"], sets[0]["u_b"], n, 0, 0, R)
        ready = [torch.cuda.Event(), torch.cuda.Event()]
        done = [torch.cuda.Event(), torch.cuda.Event()]
        for t in range(k):
            cur, nxt = t % 2, (t + 1) % 2
            # regenerate step t+1 into the other set once step t-1's gather read it
            side.wait_event(done[nxt]) if t >= 1 else side.wait_stream(main)
            with torch.cuda.stream(side):
                drivers.regen_step(sets[nxt]["u_1"], sets[nxt]["u_b"], n, t + 1, 0, R)
                ready[nxt].record(side)
            if t >= 1:
                main.wait_event(ready[cur])
            arr = dict(a, **sets[cur])
            api.adjoint_fresh(fam, n, sc, arr)
            done[cur].record(main)
        main.wait_stream(side)


def timed(fn, k):
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(main)
    fn(k)
    e.record(main)
    torch.cuda.synchronize()
    return s.elapsed_time(e) / k


res = {"serial": [], "pipelined": []}
for r in range(rounds + 1):
    for name, fn in ((("serial", serial), ("pipelined", pipelined)) if r % 2 == 0 else
                     (("pipelined", pipelined), ("serial", serial))):
        ms = timed(fn, steps)
        if r:
            res[name].append(ms)
        time.sleep(1.0)
for k, v in res.items():
    print(f"{k:10s} {statistics.median(v):.3f} ms per step  ({[round(x, 3) for x in v]})")
# the two forms compute the same c_b (bitwise): same per-step arithmetic
