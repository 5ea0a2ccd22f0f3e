"""Pin the CPU oracle restatement (oracle/sg_oracle.c) to the reference.

(1) The reference's own known-answer tests for this path
    (proj/tests/test_adjoint.cpp, test_symdiff.cpp) restated on the oracle.
(2) Golden vectors made by the UNMODIFIED reference library
    (tests/golden/make_golden.py -> oracle/_ref/ref_harness): run_nest,
    run_program and run_scatter_adjoint outputs, plus its program structure.
CPU only.
"""
import glob
import json
import os

import numpy as np
import pytest

from oracle import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def star(d):
    out = [tuple([0] * d)]
    for i in range(d):
        for s in (-1, 1):
            o = [0] * d
            o[i] = s
            out.append(tuple(o))
    return out


def dense(d):
    import itertools
    return [tuple(o) for o in itertools.product((-1, 0, 1), repeat=d)]


def count(offsets, n=16):
    d = len(offsets[0])
    nests, _ = oracle.split_offsets(sorted(offsets), [2] * d, [n - 2] * d)
    return len(nests)


def test_region_counts_match_reference_kat():
    # test_adjoint.cpp:137-151
    assert len(oracle.split_family("lap1d", 16)[0]) == 5
    assert len(oracle.split_family("wave3d", 16)[0]) == 53
    assert count(dense(2)) == 25
    assert count(dense(3)) == 125
    assert count(star(2)) == 17
    # config encodings
    assert len(oracle.split_family("wave1d", 64)[0]) == 5
    assert len(oracle.split_family("wave3d_c", 16)[0]) == 53
    assert len(oracle.split_family("burgers2d", 16)[0]) == 17
    assert len(oracle.split_family("wave3d_r4", 24)[0]) == 1457


def test_lap1d_five_regions():
    # test_adjoint.cpp:112-135 (n symbolic there; here n=16)
    nests, core = oracle.split_family("lap1d", 16)
    n = 16
    assert core == 2
    assert [ns["bounds"][0] for ns in nests] == [(0, 0), (1, 1), (2, n - 2), (n - 1, n - 1),
                                                 (n, n)]
    assert [ns["terms"] for ns in nests] == [[0], [0, 1], [0, 1, 2], [1, 2], [2]]
    assert nests[2]["core"]


def test_core_bounds_and_guards():
    # test_adjoint.cpp:96-110, :225-233
    assert oracle.core_bounds("lap1d", 16) == [(2, 14)]
    assert oracle.core_bounds("wave3d", 16) == [(2, 13)] * 3
    assert oracle.core_bounds("wave3d_r4", 768) == [(8, 759)] * 3
    assert oracle.guards_ok("wave3d", 5) and not oracle.guards_ok("wave3d", 4)
    assert oracle.guards_ok("wave3d_r4", 17) and not oracle.guards_ok("wave3d_r4", 16)
    assert oracle.guards_ok("wave1d", 5) and not oracle.guards_ok("wave1d", 4)


def test_term_order_matches_reference_active_reads():
    # test_symdiff.cpp:27-52 and the reference's structure dump
    with open(os.path.join(GOLDEN, "ref_structure.json")) as fh:
        ref = json.load(fh)
    for name in oracle.FAMILIES:
        f = oracle.family(name)
        rt = ref[name]["terms"]
        assert len(rt) == len(f.terms), name
        for (arr, off), t in zip(f.terms, rt):
            assert f.arrays[arr] == t["array"] and list(off) == t["offset"], name


@pytest.mark.parametrize("key", ["wave1d", "wave3d_c", "wave3d_c2", "burgers2d", "wave3d_r4",
                                 "lap1d", "wave3d", "burgers1d", "wave1d@16777216",
                                 "wave3d_c@512", "burgers2d@8192", "wave3d_r4@768",
                                 "wave3d_r4@1024"])
def test_nests_match_reference_structure(key):
    """Every nest's bounds, term set and core flag equal the reference's
    assemble_adjoint output (adjoint.cpp:152-163), also at the BASELINE sizes."""
    with open(os.path.join(GOLDEN, "ref_structure.json")) as fh:
        ref = json.load(fh)[key]
    name = key.split("@")[0]
    n = int(key.split("@")[1]) if "@" in key else {
        "wave1d": 64, "wave3d_c": 12, "wave3d_c2": 12, "burgers2d": 24, "wave3d_r4": 20,
        "lap1d": 16, "wave3d": 10, "burgers1d": 64}[name]
    nests, core = oracle.split_family(name, n)
    assert core == ref["core_index"]
    assert len(nests) == len(ref["nests"])
    for mine, theirs in zip(nests, ref["nests"]):
        assert [list(b) for b in mine["bounds"]] == theirs["bounds"]
        assert mine["terms"] == theirs["terms"]
        assert mine["core"] == theirs["core"]
    assert [list(b) for b in oracle.core_bounds(name, n)] == ref["core_bounds"]


def _golden_cases():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz")))


def load_golden(case):
    z = np.load(os.path.join(GOLDEN, case + ".npz"))
    name = case.rsplit("_n", 1)[0]
    n = int(case.rsplit("_n", 1)[1].split("_s")[0])
    f = oracle.family(name)
    scalars = dict(zip(f.scalars, z["scalars"].tolist()))
    grids = {k[3:]: z[k].copy() for k in z.files if k.startswith("in_")}
    adjs = {k[6:]: z[k].copy() for k in z.files if k.startswith("inadj_")}
    refs = {k[4:]: z[k] for k in z.files if k.startswith("ref_")}
    return name, n, f, scalars, grids, adjs, refs


@pytest.mark.parametrize("case", _golden_cases())
def test_oracle_matches_reference_golden(case):
    name, n, f, scalars, grids, adjs, refs = load_golden(case)
    # primal (run_nest)
    g = {k: v.copy() for k, v in grids.items()}
    assert oracle.run_primal(name, n, scalars, g) == 0
    out = f.arrays[f.output]
    assert oracle.max_rel_err(g[out], refs["primal_" + out]) <= 1e-12
    # gather (run_program), hierarchical and predicate forms, and scatter
    results = {}
    for fn in ("run_program", "run_program_predicate", "run_scatter"):
        a = {k: v.copy() for k, v in adjs.items()}
        assert getattr(oracle, fn)(name, n, scalars, {k: v.copy() for k, v in grids.items()},
                                   a) == 0
        results[fn] = a
    for i, arr in enumerate(f.arrays):
        adj = f.adjoints[i]
        if not adj or i == f.output:
            continue
        ref_g = refs["gather_" + adj]
        ref_s = refs["scatter_" + adj]
        assert oracle.max_rel_err(results["run_program"][adj], ref_g) <= 1e-12, adj
        assert oracle.max_rel_err(results["run_scatter"][adj], ref_s) <= 1e-12, adj
        # hierarchical and predicate forms are the same per-cell sequence
        assert np.array_equal(results["run_program"][adj], results["run_program_predicate"][adj])
        # the reference's own oracle-equivalence bound (interp.cpp:425)
        assert oracle.max_rel_err(ref_g, ref_s) <= 1e-12


def test_reference_verify_reports_pass():
    with open(os.path.join(GOLDEN, "ref_verify.json")) as fh:
        rep = json.load(fh)
    for k, v in rep.items():
        assert v["exit"] == 0 and v["report"]["pass"], k
