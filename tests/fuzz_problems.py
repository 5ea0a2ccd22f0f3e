"""Seeded random stencil problems for the emitter tests (test helper).

Restates the structure of the reference's fuzz generator
(proj/tests/support/problems.hpp:107-178, `random_problem`): depth d <= 3,
counters i, j, k on bounds [2, n-2], extents n+1, an active input u (and
sometimes v), an optional passive coefficient array c read at offsets in
[-1, 1], an active output r; 2-4 terms coefficient * read with read offsets
in [-2, 2], varied into max(read, 0), min(read', read), read * read' and
pow(read, 2); an optional constant; mode = or +=.  Emitted as a spec in the
reference's JSON format, so the reference's own front end (parse_spec,
validate, differentiate, assemble_adjoint) processes it.
"""
from __future__ import annotations

import random


def random_spec(seed: int, linear_only: bool = False) -> dict:
    rng = random.Random(seed)
    d = 1 + rng.randrange(3)
    counters = ["i", "j", "k"][:d]
    two_inputs = rng.randrange(3) == 0
    with_coeff = rng.randrange(2) == 0

    def idx(offs):
        out = ""
        for c, o in zip(counters, offs):
            out += f"[{c}{' + ' + str(o) if o > 0 else ' - ' + str(-o) if o < 0 else ''}]"
        return out

    def active_read():
        arr = "v" if two_inputs and rng.randrange(2) else "u"
        return arr + idx([rng.randrange(5) - 2 for _ in counters])

    def coeff_read():
        return "c" + idx([rng.randrange(3) - 1 for _ in counters])

    def coefficient():
        k = rng.randrange(3)
        if k == 0:
            return f"{1 + rng.randrange(7)}.0"
        if k == 1:
            return "a"
        return coeff_read() if with_coeff else "0.5"

    terms = []
    for _ in range(2 + rng.randrange(3)):
        read = active_read()
        term = f"{coefficient()}*{read}"
        if not linear_only:
            v = rng.randrange(5)
            if v == 0:
                term = f"{coefficient()}*max({read}, 0)"
            elif v == 1:
                term = f"{coefficient()}*min({active_read()}, {read})"
            elif v == 2:
                term = f"{read}*{active_read()}"
            elif v == 3:
                term = f"{coefficient()}*pow({read}, 2)"
        terms.append(term)
    if rng.randrange(2):
        terms.append("0.25")
    shape = ["n + 1"] * d
    arrays = {"u": {"rank": d, "shape": shape, "active": True, "adjoint": "u_b", "role": "input"}}
    if two_inputs:
        arrays["v"] = {"rank": d, "shape": shape, "active": True, "adjoint": "v_b",
                       "role": "input"}
    if with_coeff:
        arrays["c"] = {"rank": d, "shape": shape, "active": False, "role": "coefficient"}
    arrays["r"] = {"rank": d, "shape": shape, "active": True, "adjoint": "r_b", "role": "output"}
    return {
        "name": f"fuzz{seed}", "counters": counters,
        "bounds": {c: ["2", "n - 2"] for c in counters},
        "sizes": ["n"], "scalars": ["a"], "arrays": arrays,
        "lhs": "r" + "".join(f"[{c}]" for c in counters),
        "mode": "+=" if rng.randrange(2) else "=",
        "rhs": " + ".join(terms),
    }
