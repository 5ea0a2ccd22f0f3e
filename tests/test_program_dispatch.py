"""Program-keyed dispatch at the boundary (VERDICT r1 'name-keyed
dispatch'): the library matches a caller's AdjointProgram -- its canonical text
(sgb_program_family) -- against the programs its hand-tuned kernels compute,
which were exported from the reference front end (programs/<family>.canon).
A program named like a family but with another body, bounds or term list is
refused; the Python layer lowers such a program through the NVRTC emitter
(api.run_program_from) and the reference-side binding throws
stencilgrad::Error.  CPU tests need no GPU (matching is host logic); the
-m gpu tests run both routes against the reference's own run_program."""
import copy
import json
import os
import subprocess
import tempfile

import numpy as np
import pytest

from oracle import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1907_02818_b200", "libstencilgrad_b200.so")
FAMS = ("wave1d", "wave3d_c", "wave3d_c2", "burgers2d", "wave3d_r4")
needs_ref = pytest.mark.skipif(not oracle.ref_available(),
                               reason="oracle/_ref/ref_harness not built")


def _canon(f):
    with open(os.path.join(ROOT, "paper_1907_02818_b200", "programs", f + ".canon")) as fh:
        return fh.read()


def _family(text):
    from paper_1907_02818_b200 import _lib
    r = _lib.lib().sgb_program_family(text.encode())
    return None if r is None else r.decode()


@pytest.mark.parametrize("fam", FAMS)
def test_committed_programs_match_their_family(fam):
    assert _family(_canon(fam)) == fam


@pytest.mark.parametrize("fam", FAMS)
def test_edited_programs_are_refused(fam):
    from paper_1907_02818_b200 import _lib
    text = _canon(fam)
    lines = text.splitlines(keepends=True)
    edits = {
        "partial": lambda ls: [l.replace("partial ", "partial 2*", 1)
                               if l.startswith("term 0 ") else l for l in ls],
        "offset": lambda ls: [l.replace("offset -1", "offset -2", 1) for l in ls],
        "guard": lambda ls: [l.replace(">= ", ">= 1", 1) if l.startswith("guard") else l
                             for l in ls],
        "drop_nest": lambda ls: [l for i, l in enumerate(ls)
                                 if not (l.startswith("nest") and i == len(ls) - 3)],
        "core": lambda ls: ls[:-1] + ["core 0\n"],
    }
    for name, edit in edits.items():
        new = "".join(edit(list(lines)))
        if new == text:
            continue
        assert _family(new) is None, name
        assert "no hand-tuned" in _lib.lib().sgb_last_error().decode()


def test_signatures_are_the_reference_prototypes():
    """sgb_family_signature = the generated <family>_b prototype order."""
    from paper_1907_02818_b200 import _lib
    import re
    protos = json.load(open(os.path.join(ROOT, "tests", "golden", "ref_protos.json")))
    for fam in FAMS:
        sig = _lib.lib().sgb_family_signature(fam.encode()).decode()
        args = re.search(r"\((.*)\)", protos[fam]["adjoint"]).group(1).split(",")
        ints = [a.split()[-1] for a in args if a.split()[0] == "int"]
        dbls = [a.split()[-1] for a in args if a.split()[0] == "double" and "*" not in a]
        ptrs = [a.split("*")[-1].strip() for a in args if "*" in a]
        assert sig == ";".join([",".join(ints), ",".join(dbls), ",".join(ptrs)]), fam
    assert _lib.lib().sgb_family_signature(b"lap1d") is None


@needs_ref
@pytest.mark.parametrize("spec", ["wave1d", "wave3d_c", "wave3d_c2", "burgers2d", "wave3d_r4"])
def test_reference_programs_match_through_the_binding(spec):
    """The binding's canonical text of the reference's own assemble_adjoint
    (ref_harness match) selects the family; the bundled examples select none."""
    r = subprocess.run([oracle.ref_harness_path(), "match", oracle.spec_path(spec)],
                       capture_output=True, text=True, env=dict(os.environ, SGB_LIB=LIB),
                       timeout=60)
    assert r.returncode == 0, r.stderr
    assert json.loads(r.stdout)["family"] == spec


def _modified_r4(tmp):
    """A Problem NAMED wave3d_r4 whose rhs differs (one 8th-order weight)."""
    spec = json.load(open(oracle.spec_path("wave3d_r4")))
    assert "1.6*u_1[i-1][j][k]" in spec["rhs"]
    spec["rhs"] = spec["rhs"].replace("1.6*u_1[i-1][j][k]", "1.5*u_1[i-1][j][k]", 1)
    path = os.path.join(tmp, "wave3d_r4_mod.json")
    json.dump(spec, open(path, "w"))
    return spec, path


@needs_ref
def test_modified_program_named_like_a_family_is_refused(tmp_path):
    _, path = _modified_r4(str(tmp_path))
    r = subprocess.run([oracle.ref_harness_path(), "match", path], capture_output=True,
                       text=True, env=dict(os.environ, SGB_LIB=LIB), timeout=60)
    assert r.returncode == 0, r.stderr
    rep = json.loads(r.stdout)
    assert rep["name"] == "wave3d_r4" and rep["family"] is None
    assert "wave3d_r4" in rep["why"]
    for ex in ("example:lap1d", "example:wave3d", "example:burgers1d"):
        r = subprocess.run([oracle.ref_harness_path(), "match", ex], capture_output=True,
                           text=True, env=dict(os.environ, SGB_LIB=LIB), timeout=60)
        assert json.loads(r.stdout)["family"] is None, ex


def test_python_program_matching():
    from paper_1907_02818_b200 import api
    for fam in FAMS:
        assert api.program_family(api.load_program(fam)) == fam
    prog = api.load_program("wave3d_r4")
    mod = copy.deepcopy(prog)
    mod["spec"]["rhs"] = mod["spec"]["rhs"].replace("1.6*", "1.5*", 1)
    assert api.program_family(mod) is None
    mod = copy.deepcopy(prog)
    mod["terms"][3]["partial"] = "2*" + mod["terms"][3]["partial"]
    assert api.program_family(mod) is None
    assert api.program_family(api.load_program("lap1d")) is None


@pytest.mark.gpu
@needs_ref
def test_binding_refuses_modified_program_on_gpu(tmp_path):
    """ref_harness b200: the binding throws for the modified program (exit 3)
    instead of running the hard-coded stencil."""
    _, path = _modified_r4(str(tmp_path))
    n = 20
    rng = np.random.default_rng(3)
    with tempfile.TemporaryDirectory() as td:
        for k in ("c", "c_b", "u_1", "u_1_b", "u_b"):
            rng.standard_normal((n, n, n)).tofile(os.path.join(td, k + ".f64"))
        r = subprocess.run([oracle.ref_harness_path(), "b200", path, str(n), td, "D=0.01"],
                           capture_output=True, text=True, env=dict(os.environ, SGB_LIB=LIB),
                           timeout=120)
    assert r.returncode == 3, r.stdout + r.stderr
    assert "no B200 kernel" in json.loads(r.stdout)["error"]


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("which", ["family", "modified"])
def test_run_program_from_matches_reference(tmp_path, which):
    """api.run_program_from(program): the family's own program runs the
    hand-tuned kernels, the modified one the NVRTC emitter; both equal the
    reference's run_program on the same Env at 1e-12 (fp64)."""
    from paper_1907_02818_b200 import api
    n = 20
    if which == "family":
        spec, path = json.load(open(oracle.spec_path("wave3d_r4"))), oracle.spec_path("wave3d_r4")
    else:
        spec, path = _modified_r4(str(tmp_path))
    r = subprocess.run([oracle.ref_harness_path(), "spec", path], capture_output=True,
                       text=True, timeout=60)
    spec = json.loads(r.stdout)
    info = json.loads(subprocess.run([oracle.ref_harness_path(), "info", path, str(n)],
                                     capture_output=True, text=True, timeout=60).stdout)
    program = {"spec": spec, "terms": info["terms"]}
    assert (api.program_family(program) is not None) == (which == "family")
    rng = np.random.default_rng(5)
    grids = {k: rng.standard_normal((n, n, n)) for k in ("c", "u_1", "u_2", "u")}
    grids["c"] = rng.uniform(1.5, 4.5, (n, n, n))
    adjs = {k: rng.standard_normal((n, n, n)) for k in ("c_b", "u_1_b", "u_b")}
    got, route = api.run_program_from(program, {"n": n}, {"D": 0.01}, grids, adjs,
                                      return_route=True)
    assert route == ("hand-tuned" if which == "family" else "emitter")
    with tempfile.TemporaryDirectory() as td, tempfile.TemporaryDirectory() as od:
        for k, v in {**grids, **adjs}.items():
            v.tofile(os.path.join(td, k + ".f64"))
        rr = subprocess.run([oracle.ref_harness_path(), "run", path, str(n), td, od, "D=0.01"],
                            capture_output=True, text=True, timeout=300)
        assert rr.returncode == 0, rr.stderr
        for k in ("c_b", "u_1_b"):
            want = np.fromfile(os.path.join(od, "gather_" + k + ".f64")).reshape(n, n, n)
            assert oracle.max_rel_err(got[k], want) <= 1e-12, k
