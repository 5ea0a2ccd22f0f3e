"""Seeded host-side inputs with the BASELINE.json distributions (test helper).

Used by the golden-fixture generator and the parity tests at oracle-sized n.
(The benchmark generates its full-size inputs on the device with the product's
counter-based generators; see paper_1907_02818_b200/csrc/inputs.cu and drivers.py.)

Distributions (BASELINE.json ``configs``):
  wave1d     u, u_prev, u_next_b ~ N(0,1), zero Dirichlet ends; c ~ U[1.5,4.5]; D=0.25
  wave3d_c*  u_1, u_2, u_b ~ N(0,1), 1-point zero halo; c ~ U[1.5,4.5]; D=0.1
  burgers2d  u ~ U[-1,1] smoothed by 3 interior passes of a 5-point average;
             u_b ~ N(0,1); C=0.2, D=nu*C=0.002
  wave3d_r4  c ~ U[1.5,4.5] constant on 8 equal layers along i; u_1, u_2, u_b ~ N(0,1),
             4-point zero halo; D=0.01
"""
from __future__ import annotations

import numpy as np

SCALARS = {
    "wave1d": {"D": 0.25},
    "wave3d_c": {"D": 0.1},
    "wave3d_c2": {"D": 0.1},
    "wave3d": {"D": 0.1},
    "burgers2d": {"C": 0.2, "D": 0.002},
    "wave3d_r4": {"D": 0.01},
    "lap1d": {},
    "burgers1d": {"C": 0.3, "D": 0.05},
}


def zero_halo(a: np.ndarray, h: int) -> np.ndarray:
    if h <= 0:
        return a
    for ax in range(a.ndim):
        idx = [slice(None)] * a.ndim
        idx[ax] = slice(0, h)
        a[tuple(idx)] = 0.0
        idx[ax] = slice(a.shape[ax] - h, None)
        a[tuple(idx)] = 0.0
    return a


def smooth5(u: np.ndarray, passes: int = 3) -> np.ndarray:
    """(u + 4 neighbours) / 5 on the interior only, boundary ring untouched."""
    for _ in range(passes):
        v = u.copy()
        v[1:-1, 1:-1] = (u[1:-1, 1:-1] + u[:-2, 1:-1] + u[2:, 1:-1] + u[1:-1, :-2]
                         + u[1:-1, 2:]) / 5.0
        u = v
    return u


def layered_c(n: int, rng: np.random.Generator, layers: int = 8) -> np.ndarray:
    vals = rng.uniform(1.5, 4.5, size=layers)
    lay = (np.arange(n) * layers) // n
    return np.broadcast_to(vals[lay][:, None, None], (n, n, n)).copy()


def family_inputs(name: str, n: int, seed: int, accumulate: bool = False, ties: bool = True):
    """Returns (scalars, grids, adjs) as float64 arrays keyed by the spec names.

    accumulate=True gives the input adjoints random initial values so that the
    ``+=`` contract is exercised; otherwise they start at zero as
    in make_env (interp.cpp:280-286).
    """
    rng = np.random.default_rng(seed)
    N = rng.standard_normal
    U = rng.uniform
    sc = dict(SCALARS[name])
    g: dict = {}
    a: dict = {}
    if name == "wave1d":
        g["c"] = U(1.5, 4.5, n)
        g["u"] = zero_halo(N(n), 1)
        g["u_prev"] = zero_halo(N(n), 1)
        g["u_next"] = N(n)
        a["u_next_b"] = N(n)
        for k in ("c_b", "u_b", "u_prev_b"):
            a[k] = N(n) if accumulate else np.zeros(n)
    elif name in ("wave3d_c", "wave3d_c2", "wave3d"):
        s = (n, n, n)
        g["c"] = U(1.5, 4.5, s)
        g["u_1"] = zero_halo(N(s), 1)
        g["u_2"] = zero_halo(N(s), 1)
        g["u"] = N(s)
        a["u_b"] = N(s)
        ks = ["u_1_b", "u_2_b"] + ([] if name == "wave3d" else ["c_b"])
        for k in ks:
            a[k] = N(s) if accumulate else np.zeros(s)
    elif name == "burgers2d":
        s = (n, n)
        u = smooth5(U(-1.0, 1.0, s))
        if ties:  # exact zeros exercise the >= tie rule (symdiff.cpp:269-274)
            idx = rng.integers(0, n, size=(max(2, n // 4), 2))
            u[idx[:, 0], idx[:, 1]] = 0.0
            u[n // 2, :3] = -0.0
        g["u_1"] = u
        g["u"] = N(s)
        a["u_b"] = N(s)
        a["u_1_b"] = N(s) if accumulate else np.zeros(s)
    elif name == "wave3d_r4":
        s = (n, n, n)
        g["c"] = layered_c(n, rng)
        g["u_1"] = zero_halo(N(s), 4)
        g["u_2"] = zero_halo(N(s), 4)
        g["u"] = N(s)
        a["u_b"] = N(s)
        for k in ("c_b", "u_1_b"):
            a[k] = N(s) if accumulate else np.zeros(s)
    elif name == "lap1d":
        g["c"] = U(1.5, 4.5, n + 1)
        g["u"] = N(n + 1)
        g["r"] = N(n + 1)
        a["rb"] = N(n + 1)
        a["ub"] = N(n + 1) if accumulate else np.zeros(n + 1)
    elif name == "burgers1d":
        u = U(-1.0, 1.0, n)
        if ties:
            u[n // 3] = 0.0
        g["u_1"] = u
        g["u"] = N(n)
        a["u_b"] = N(n)
        a["u_1_b"] = N(n) if accumulate else np.zeros(n)
    else:
        raise KeyError(name)
    return sc, g, a
