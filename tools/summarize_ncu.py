"""Key metrics + hottest source lines of an `ncu --set full --import-source on`
report, as markdown.  Usage: python tools/summarize_ncu.py <rep> <out.md> [title]"""
import collections
import csv
import io
import subprocess
import sys

rep, out_path = sys.argv[1], sys.argv[2]
title = sys.argv[3] if len(sys.argv) > 3 else rep
KEYS = ["Duration", "Elapsed Cycles", "SM Frequency", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "Theoretical Occupancy", "Achieved Occupancy", "Warp Cycles Per Issued Instruction",
        "Avg. Active Threads Per Warp", "No Eligible", "Block Limit Registers", "Block Limit Shared Mem"]
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(det)))
h = rows[0]
ki, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
per = collections.OrderedDict()
for r in rows[1:]:
    if len(r) > vi and r[mi] in KEYS:
        per.setdefault(r[ki].split("(")[0], collections.OrderedDict())[r[mi]] = f"{r[vi]} {r[ui]}".strip()
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
dram = {}
if rr:
    hh = rr[0]
    try:
        kk = hh.index("Kernel Name")
        cols = [hh.index(c) for c in ("dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum")]
        for r in rr[2:]:
            dram[r[kk].split("(")[0]] = [r[c] + " " + rr[1][c] for c in cols]
    except ValueError:
        pass
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
funcs = {}
cur_f = cur = fname = None
hdr = None
for r in csv.reader(io.StringIO(src)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        cur_f = r[1].split("(")[0]
        funcs.setdefault(cur_f, collections.defaultdict(lambda: [0.0, 0.0, ""]))
        continue
    if r[0] == "Line No":
        hdr = r
        ie, st = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if r[0] != "" and hdr and len(r) > ie and cur_f:
        # line rows carry the per-line aggregates; the SASS rows below repeat them
        try:
            key = (fname, r[0], r[1].strip()[:80])
            funcs[cur_f][key][0] += float(r[ie] if r[ie] not in ("-", "") else 0)
            funcs[cur_f][key][1] += float(r[st] if r[st] not in ("-", "") else 0)
        except ValueError:
            pass
lines = [f"# {title}", ""]
for k, m in per.items():
    lines += [f"## {k}", "", "| metric | value |", "|---|---|"] + [f"| {a} | {b} |" for a, b in m.items()]
    if k in dram:
        lines.append(f"| dram__bytes_read.sum / write.sum / smsp__inst_executed.sum | {' / '.join(dram[k])} |")
    fk = [f for f in funcs if f.endswith(k.split("::")[-1]) or f == k]
    if fk:
        agg = funcs[fk[0]]
        ti = sum(v[0] for v in agg.values()) or 1
        ts = sum(v[1] for v in agg.values()) or 1
        lines += ["", "Hottest source lines (share of warp-stall samples / executed instructions):", "",
                  "| stall % | inst % | line | source |", "|---|---|---|---|"]
        for (f, ln, s), v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:12]:
            lines.append(f"| {v[1] / ts * 100:.1f} | {v[0] / ti * 100:.1f} | {f}:{ln} | `{s}` |")
    lines.append("")
open(out_path, "w").write("\n".join(lines) + "\n")
print("\n".join(lines[:60]))
