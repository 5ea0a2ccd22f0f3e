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
    # the canonical program text the B200 library matches callers against
    # (b200_program_text; embedded by build.py, csrc/programs.cu)
    with open(os.path.join(HERE, name + ".canon"), "w") as fh:
        fh.write(run("canon", sp))
    print(name, len(info["terms"]), "terms")

# <family>_b's generated prototype (sizes; scalars; arrays), from the C the
# reference emitted itself (oracle/_ref/gen/<family>_protos.h)
import re  # noqa: E402
sigs = {}
for name in ["wave1d", "wave3d_c", "wave3d_c2", "burgers2d", "wave3d_r4"]:
    text = open(os.path.join(oracle.REF_DIR, "gen", name + "_protos.h")).read()
    args = re.search(r"int\s+" + name + r"_b\(([^)]*)\)", text).group(1).split(",")
    ints, dbls, ptrs = [], [], []
    for a in args:
        a = a.replace("*", " ").split()
        (ptrs if len(a) > 2 else ints if a[0] == "int" else dbls).append(a[-1])
    sigs[name] = ";".join([",".join(ints), ",".join(dbls), ",".join(ptrs)])
with open(os.path.join(HERE, "signatures.json"), "w") as fh:
    json.dump(sigs, fh, indent=1)
print(sigs)
