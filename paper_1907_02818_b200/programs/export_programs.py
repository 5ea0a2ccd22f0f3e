"""Export the reference front end's output for each family as {spec, terms}.

The reference's compile-time tool (parse_spec -> validate -> differentiate ->
assemble_adjoint) runs once on the host; like its emitted C, its output is an
artefact the back end consumes.  Run in the build container (needs
oracle/_ref/ref_harness, built from /root/reference):

    python paper_1907_02818_b200/programs/export_programs.py
"""
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from oracle import oracle  # noqa: E402  (build-time only)

for name in ["wave1d", "wave3d_c", "wave3d_c2", "burgers2d", "wave3d_r4", "lap1d", "wave3d",
             "burgers1d"]:
    sp = oracle.spec_path(name)
    run = lambda *a: subprocess.run([oracle.ref_harness_path(), *a], check=True,
                                    capture_output=True, text=True).stdout
    spec = json.loads(run("spec", sp))
    info = json.loads(run("info", sp, "64"))
    with open(os.path.join(HERE, name + ".json"), "w") as fh:
        json.dump({"spec": spec, "terms": info["terms"],
                   "source": "reference front end (ref_harness spec/info: serialize_spec, "
                             "assemble_adjoint terms with to_input_string partials)"},
                  fh, indent=1)
    print(name, len(info["terms"]), "terms")
