"""Emitted stream form vs the flat form (developer aid): agreement to
rounding (NaN sentinel cells untouched) on the 3D families at several sizes.
python scripts/stream_check.py"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1907_02818_b200 import emitter  # noqa: E402

for fam in ["wave3d_r4", "wave3d_c", "wave3d_c2", "wave3d"]:
    for dt in ("f64", "f32"):
        ep = emitter.load_program(fam, dt)
        for n in (20, 68, 100):
            sizes = {"n": n}
            rng = np.random.default_rng(n)
            td = torch.float64 if dt == "f64" else torch.float32
            base = {}
            for arr in ep.param_arrays():
                shp = tuple(ep._eval_aff(a, sizes) for a in ep._shape_of(arr))
                v = rng.standard_normal(shp)
                if arr.endswith("_b") and arr != ep.seed:
                    v.reshape(-1)[::7] = np.nan
                base[arr] = torch.from_numpy(v).to(td).cuda()
            a = {k: v.clone() for k, v in base.items()}
            b = {k: v.clone() for k, v in base.items()}
            sc = {s: 0.3 for s in ep.scalars}
            ep.adjoint(sizes, sc, a, form="stream")
            ep.adjoint(sizes, sc, b, form="flat")
            torch.cuda.synchronize()
            for t in sorted({t.adjoint for t in ep.terms}):
                x, y = a[t].double(), b[t].double()
                same_nan = torch.equal(torch.isnan(x), torch.isnan(y))
                m = ~torch.isnan(y)
                err = float(((x[m] - y[m]).abs() / (1 + y[m].abs())).max())
                print(f"{fam} {dt} n={n} {t}: NaN cells same {same_nan}, max rel {err:.2e}",
                      flush=True)
