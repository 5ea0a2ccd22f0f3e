"""Summarise an ncu report: key throughput metrics, stall mix, top stalled SASS lines."""
import csv
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr = rows[0]
for vals in rows[2:]:
    get = {h: vals[i] for i, h in enumerate(hdr)}
    print("kernel:", get.get("Kernel Name", "?")[:90])
    for w in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
              "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
              "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
              "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
              "smsp__issue_active.avg.pct_of_peak_sustained_active",
              "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
              "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
              "lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum",
              "lts__t_sector_hit_rate.pct", "sm__cycles_elapsed.avg.per_second"]:
        if w in get:
            print(f"  {w:60s} {get[w]}")
    items = [(float(v), h) for h, v in get.items()
             if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")
             and v.replace(".", "").isdigit()]
    tot = sum(v for v, _ in items) or 1
    for v, h in sorted(items, reverse=True)[:8]:
        print(f"  {v / tot * 100:5.1f}% {h[len('smsp__pcsamp_warps_issue_stalled_'):]}")
if len(sys.argv) > 2:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "sass"], capture_output=True, text=True).stdout
    # one section per kernel: a "Kernel Name" line, a header line, then rows;
    # argv[3] (optional) selects the sections whose kernel name contains it
    want = sys.argv[3] if len(sys.argv) > 3 else None
    h, data, keep = None, [], True
    for x in csv.reader(src.splitlines()):
        if x and x[0] == "Kernel Name":
            keep = want is None or want in x[1]
            h = None
            continue
        if x and x[0] == "Address":
            h = x
            iS = h.index("Warp Stall Sampling (All Samples)")
            iE = h.index("Instructions Executed")
            iSrc = h.index("Source")
            continue
        if keep and h and len(x) == len(h):
            data.append(x)
    tot = sum(float(x[iS] or 0) for x in data)
    totE = sum(float(x[iE] or 0) for x in data)
    c, s = Counter(), Counter()
    for x in data:
        toks = x[iSrc].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") else toks[0]
        op = op.split(".")[0]
        c[op] += float(x[iE] or 0)
        s[op] += float(x[iS] or 0)
    print("  opcode mix (exec%, stall%):")
    for op, v in c.most_common(16):
        print(f"    {op:10s} {v / totE * 100:5.1f}% {s[op] / tot * 100:5.1f}%")
    print("  top stalled:")
    for x in sorted(data, key=lambda x: -float(x[iS] or 0))[:int(sys.argv[2])]:
        print("   ", x[iS], x[iE], x[iSrc][:80])
