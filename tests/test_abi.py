"""C-ABI boundary checks that run without a GPU.

* the library builds for sm_100a and loads;
* it exports every symbol include/stencilgrad_b200.h declares;
* each generated-function entry point keeps the reference emitter's
  parameter order (codegen.cpp:198-230), checked against the prototypes the
  unmodified reference emits for the same specs (tests/golden/ref_protos.json);
* the cubin really targets sm_100a and the hot kernel uses TMA (UTMALDG).
"""
import json
import os
import re
import subprocess

import pytest

from paper_1907_02818_b200 import _lib, build

HERE = os.path.dirname(__file__)


@pytest.fixture(scope="module")
def lib():
    build.build()
    return _lib.lib()


def test_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    declared = set(_lib.PROTOTYPES)
    assert declared, "header parse found no prototypes"
    missing = declared - exported
    assert not missing, f"declared but not exported: {sorted(missing)}"
    for name in declared:
        assert getattr(lib, name) is not None


def test_parameter_order_matches_reference_emitter():
    with open(os.path.join(HERE, "golden", "ref_protos.json")) as fh:
        ref = json.load(fh)
    for fam, protos in ref.items():
        for kind, proto in protos.items():
            name = fam + {"primal": "", "adjoint": "_b", "scatter": "_scatter_b"}[kind]
            ref_params = re.findall(r"(\w+)\s*(?:,|\))", proto.split("(", 1)[1])
            for sfx in ("f32", "f64"):
                _, params = _lib.PROTOTYPES[f"{name}_{sfx}"]
                mine = [p for _, p in params][:-1]  # drop trailing stream
                assert mine == ref_params, (name, sfx, mine, ref_params)


def test_no_device_call_without_gpu_is_needed_to_load(lib):
    assert lib.sgb_version().startswith(b"stencilgrad_b200")
    assert lib.sgb_launch_count() == 0


def test_guard_and_einval_paths_without_gpu(lib):
    # host-side checks fire before any launch (no GPU needed)
    assert lib.wave3d_r4_b_f32(16, 0.01, None, None, None, None, None, None) == _lib.SGB_GUARD
    assert lib.wave3d_r4_b_f32(32, 0.01, None, None, None, None, None, None) == _lib.SGB_EINVAL
    assert lib.wave1d_b_f64(4, 0.25, None, None, None, None, None, None, None) == _lib.SGB_GUARD
    assert lib.burgers2d_b_f64(0, 0.2, 0.002, None, None, None, None) == _lib.SGB_EINVAL


def test_sass_is_sm100a_with_tma():
    r = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", _lib.LIB_PATH],
                       capture_output=True, text=True)
    assert r.returncode == 0
    assert "sm_100a" in r.stdout
    sass = r.stdout
    i = sass.find("star3_tma_kernel")
    assert i >= 0
    assert "UTMALDG" in sass, "TMA loads missing from the streaming kernel"


def test_missing_entry_kind_raises_stencil_error():
    """An entry the header does not declare (fresh_u2 is radius-1 fp32 only)
    is a StencilError naming the missing function, not a KeyError."""
    from paper_1907_02818_b200 import api
    assert api.function_name("wave3d_c", "fresh_u2", "f32") == "wave3d_c_b_fresh_u2_f32"
    for fam, kind, dt in [("wave3d_r4", "fresh_u2", "f32"), ("wave3d_c", "fresh_u2", "f64"),
                          ("wave1d", "fresh", "f64"), ("wave3d_r4", "bogus", "f32")]:
        with pytest.raises(_lib.StencilError):
            api.function_name(fam, kind, dt)
        with pytest.raises(_lib.StencilError):
            api.array_params(fam, kind, dt)
