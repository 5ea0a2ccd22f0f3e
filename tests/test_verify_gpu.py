"""Device-side parity reductions (sgb_compare_*, sgb_dot_*) against numpy:
the reference's compare_grids metric (interp.cpp:290-298) and the dot
products of dot_product_test (interp.cpp:354-375)."""
import numpy as np
import pytest

from oracle import oracle

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("count", [0, 1, 1000, 3 * 2 ** 20 + 7])
@pytest.mark.parametrize("dt", ["f32", "f64"])
def test_compare_and_dot_match_numpy(count, dt):
    import torch
    from paper_1907_02818_b200 import api
    rng = np.random.default_rng(count)
    b = rng.standard_normal(count) * 10
    a = b + rng.standard_normal(count) * 1e-3
    td = torch.float32 if dt == "f32" else torch.float64
    ta = torch.from_numpy(a).to("cuda", td)
    tb = torch.from_numpy(b).to("cuda")
    got = api.compare(ta, tb)
    a_r = ta.double().cpu().numpy()
    if count:
        assert got["max_rel"] == pytest.approx(oracle.max_rel_err(a_r, b), rel=1e-12)
        assert got["norm_rel"] == pytest.approx(oracle.norm_rel_err(a_r, b), rel=1e-9)
    else:
        assert got["max_rel"] == 0.0
    assert got["nonfinite"] == 0
    d = api.dot(ta, ta)
    assert d == pytest.approx(float(np.dot(a_r, a_r)), rel=1e-12, abs=1e-300)
    # deterministic
    assert api.compare(ta, tb) == got


def test_compare_counts_nonfinite():
    import torch
    from paper_1907_02818_b200 import api
    a = torch.zeros(100, device="cuda")
    b = torch.zeros(100, device="cuda", dtype=torch.float64)
    a[3] = float("nan")
    a[7] = float("inf")
    r = api.compare(a, b)
    assert r["nonfinite"] == 2 and r["max_rel"] == 0.0
