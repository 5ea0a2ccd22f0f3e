"""Generate the golden fixtures under tests/golden/ from the UNMODIFIED reference.

Run in the build container (it needs /root/reference and oracle/_ref, built by
``make -C oracle/ref``):

    python tests/golden/make_golden.py

For each family it draws seeded inputs with the BASELINE.json distributions
(scaled down to a size the reference interpreter finishes in seconds), writes
them as raw fp64, runs ``oracle/_ref/ref_harness run`` -- i.e. the reference's
own ``run_nest`` / ``run_program`` / ``run_scatter_adjoint``
(interp.cpp:183-228) -- and stores inputs + outputs in ``<family>_n<N>.npz``.
It also stores the reference's program structure (``ref_harness info``:
terms, partials, nest bounds/term sets, core bounds, guards) as JSON, and the
reference's own ``verify_problem`` reports for the SPEC acceptance cases
(SPEC.md:473-474).  The fixtures are committed; this script is how they were
made.  Nothing on the GPU box reads /root/reference.
"""
from __future__ import annotations

import json
import os
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle  # noqa: E402
from tests import inputs as gen  # noqa: E402

# family -> (n, seed).  Sizes keep the reference interpreter (~2-9 us/pt) fast.
CASES = {
    "wave1d": [(64, 0), (5, 1)],
    "wave3d_c": [(12, 0), (5, 3)],
    "wave3d_c2": [(12, 0)],
    "burgers2d": [(24, 0), (5, 2)],
    "wave3d_r4": [(20, 0), (17, 5)],
    "lap1d": [(16, 0)],
    "wave3d": [(10, 0)],
    "burgers1d": [(64, 0)],
}
INFO_SIZES = {"wave1d": 64, "wave3d_c": 12, "wave3d_c2": 12, "burgers2d": 24, "wave3d_r4": 20,
              "lap1d": 16, "wave3d": 10, "burgers1d": 64}


MAKE_ENV_CASES = [("wave1d", 256, 7), ("wave3d_c", 16, 7), ("wave3d_c2", 12, 3),
                  ("burgers2d", 64, 7), ("wave3d_r4", 24, 7), ("wave3d_r4", 20, 0)]


def harness(*args) -> str:
    r = subprocess.run([oracle.ref_harness_path(), *map(str, args)], check=True,
                       capture_output=True, text=True)
    return r.stdout


def make_case(name: str, n: int, seed: int) -> str:
    f = oracle.family(name)
    scalars, grids, adjs = gen.family_inputs(name, n, seed, accumulate=True)
    with tempfile.TemporaryDirectory() as tin, tempfile.TemporaryDirectory() as tout:
        for k, v in {**grids, **adjs}.items():
            v.astype(np.float64).tofile(os.path.join(tin, k + ".f64"))
        harness("run", oracle.spec_path(name), n, tin, tout,
                *[f"{k}={v!r}" for k, v in scalars.items()])
        out = {}
        shape = f.shape(n)
        for fn in os.listdir(tout):
            out["ref_" + fn[:-4]] = np.fromfile(os.path.join(tout, fn)).reshape(shape)
    payload = {"in_" + k: v for k, v in grids.items()}
    payload.update({"inadj_" + k: v for k, v in adjs.items()})
    payload.update(out)
    payload["scalars"] = np.array([scalars[s] for s in f.scalars], dtype=np.float64)
    path = os.path.join(HERE, f"{name}_n{n}_s{seed}.npz")
    np.savez_compressed(path, **payload)
    return path


def main() -> None:
    if not oracle.ref_available():
        raise SystemExit("oracle/_ref/ref_harness missing: run make -C oracle/ref")
    for name, cases in CASES.items():
        for n, seed in cases:
            print("golden", make_case(name, n, seed))
    info = {name: json.loads(harness("info", oracle.spec_path(name), n))
            for name, n in INFO_SIZES.items()}
    # structure at the full BASELINE sizes too (nest counts do not depend on n,
    # bounds do)
    for name, n in [("wave1d", 1 << 24), ("wave3d_c", 512), ("burgers2d", 8192),
                    ("wave3d_r4", 768), ("wave3d_r4", 1024)]:
        info[f"{name}@{n}"] = json.loads(harness("info", oracle.spec_path(name), n))
    with open(os.path.join(HERE, "ref_structure.json"), "w") as fh:
        json.dump(info, fh, indent=0)
    # verify_problem on the SPEC acceptance cases and the config encodings
    verify = {}
    for name, n, seed in [("wave3d", 16, 7), ("burgers1d", 256, 7), ("wave1d", 256, 7),
                          ("wave3d_c", 16, 7), ("burgers2d", 64, 7), ("wave3d_r4", 24, 7)]:
        r = subprocess.run([oracle.ref_harness_path(), "verify", oracle.spec_path(name), str(n),
                            str(seed), "2"], capture_output=True, text=True)
        verify[f"{name}_n{n}_s{seed}"] = {"exit": r.returncode, "report": json.loads(r.stdout)}
    with open(os.path.join(HERE, "ref_verify.json"), "w") as fh:
        json.dump(verify, fh, indent=1)
    # make_env digests (scalars, per-grid sums and samples): pins sgb::make_env
    envs = {}
    for name, n, seed in MAKE_ENV_CASES:
        envs[f"{name}_n{n}_s{seed}"] = json.loads(
            harness("makeenv", oracle.spec_path(name), n, seed))
    with open(os.path.join(HERE, "ref_make_env.json"), "w") as fh:
        json.dump(envs, fh, indent=1)
    # the reference emitter's prototypes (emit_primal/_adjoint/_scatter_adjoint
    # with restrict, as cmd_bench; codegen.cpp:213-230) -- the C-ABI parameter order
    protos = {}
    with tempfile.TemporaryDirectory() as td:
        for name in ("wave1d", "wave3d_c", "wave3d_c2", "burgers2d", "wave3d_r4"):
            harness("emit", oracle.spec_path(name), td)
            lines = open(os.path.join(td, name + "_protos.h")).read().splitlines()
            protos[name] = {k: v.replace("restrict ", "") for k, v in
                            zip(("primal", "adjoint", "scatter"), lines)}
    with open(os.path.join(HERE, "ref_protos.json"), "w") as fh:
        json.dump(protos, fh, indent=1)
    print("structure + verify + protos written")


if __name__ == "__main__":
    main()
