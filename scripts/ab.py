"""A/B of a kernel under run-time knobs (developer aid): each variant runs in
its own process (env set), prints its median time over 30 back-to-back-timed
calls and a bitwise digest of the outputs, so variants that only change
scheduling can be checked for identical results.  Usage:
    python scripts/ab.py [n] [fam=wave3d_r4] [kind=primal|adjoint] "" "SGB_ICHUNKS=4" ...
"""
import os
import subprocess
import sys

CHILD = r"""
import os, sys, torch
sys.path.insert(0, ".")
from paper_1907_02818_b200 import api
from scripts.quick_time import time_it
n = int(sys.argv[1]); fam = sys.argv[2]; kind = sys.argv[3]
g = torch.Generator(device="cuda"); g.manual_seed(0)
names = api.array_params(fam, kind)
dt = torch.float64 if os.environ.get("AB_F64") else torch.float32
a = {nm: torch.randn((n, n, n), device="cuda", generator=g, dtype=dt) for nm in names}
sc = {"D": 0.01 if fam == "wave3d_r4" else 0.1}
fn = getattr(api, "primal" if kind == "primal" else "adjoint")
ms = time_it(lambda: fn(fam, n, sc, a), iters=30, warm=5)
import hashlib
outs = [names[-1]] if kind == "primal" else [x for x in names if x.endswith("_b") and x != "u_b"]
if kind == "adjoint":   # digest one call from zeroed accumulators
    for nm in outs:
        a[nm].zero_()
fn(fam, n, sc, a); torch.cuda.synchronize()
hh = hashlib.sha1()
for nm in outs:
    hh.update(a[nm].cpu().numpy().tobytes())
h = hh.hexdigest()[:16]
print(f"RESULT {ms:.4f} {h}")
"""


def main():
    args = sys.argv[1:]
    n = 768
    fam = "wave3d_r4"
    kind = "primal"
    if args and args[0].isdigit():
        n = int(args.pop(0))
    if args and args[0].startswith("fam="):
        fam = args.pop(0)[4:]
    if args and args[0].startswith("kind="):
        kind = args.pop(0)[5:]
    bpp = {"primal": 16, "adjoint": {"wave3d_r4": 28}.get(fam, 36)}[kind]
    if os.environ.get("AB_F64"):
        bpp *= 2
    variants = args or [""]
    for v in variants:
        env = dict(os.environ)
        for kv in v.split():
            k, val = kv.split("=", 1)
            env[k] = val
        r = subprocess.run([sys.executable, "-c", CHILD, str(n), fam, kind], env=env,
                           capture_output=True, text=True)
        line = [x for x in r.stdout.splitlines() if x.startswith("RESULT")]
        if not line:
            print(f"{v or 'default':40s} FAILED\n{r.stderr[-800:]}", flush=True)
            continue
        _, ms, h = line[0].split()
        pts = n ** 3
        print(f"{v or 'default':40s} {float(ms):7.3f} ms  {pts * bpp / float(ms) / 1e6:6.0f} GB/s  "
              f"digest {h}", flush=True)


if __name__ == "__main__":
    main()
