"""Executed-SASS opcode mix per kernel of an ncu report (needs -lineinfo and
--import-source / --set full): python scripts/sass_mix.py rep.ncu-rep [top]"""
import collections
import csv
import re
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
text = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                      capture_output=True, text=True).stdout
kern, hdr, data = None, None, collections.defaultdict(list)
for r in csv.reader(text.splitlines()):
    if not r:
        continue
    if r[0] == "Kernel Name":
        kern = r[1][:70]
        continue
    if r[0] == "Address":
        hdr = r
        continue
    if hdr and kern:
        data[kern].append(dict(zip(hdr, r)))
for k, ins in data.items():
    op, tot = collections.Counter(), 0
    for d in ins:
        n = int(d.get("Instructions Executed") or 0)
        tot += n
        m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?", d["Source"])
        if m:
            op[m.group(2) + (m.group(3) or "")[:12]] += n
    print(f"{k}: {tot:.4e} warp instructions executed")
    for o, n in op.most_common(top):
        print(f"   {o:28s} {n:.3e} {100 * n / max(tot, 1):5.1f}%")
