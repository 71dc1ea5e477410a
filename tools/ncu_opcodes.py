"""Executed SASS instructions per opcode for one kernel of an ncu report
(--import-source on).  Usage: python tools/ncu_opcodes.py <rep> <kernel-substring> [top]"""
import collections
import csv
import io
import subprocess
import sys

rep, want = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
hdr, func = None, ""
ops, stall = collections.Counter(), collections.Counter()
for r in csv.reader(io.StringIO(src)):
    if not r:
        continue
    if r[0] in ("Function Name", "Kernel Name"):
        func = r[1]
        continue
    if r[0] == "Address":
        hdr = r
        continue
    if hdr is None or want not in func:
        continue
    d = dict(zip(hdr, r))
    text = d.get("Source", "").strip().split()
    if not text:
        continue
    op = text[1] if text[0].startswith("@") and len(text) > 1 else text[0]
    op = op.split(".")[0]
    try:
        ops[op] += float(d["Instructions Executed"])
        stall[op] += float(d["Warp Stall Sampling (All Samples)"])
    except (KeyError, ValueError):
        pass
T, S = sum(ops.values()) or 1, sum(stall.values()) or 1
print(f"{want}: {T:.3g} warp instructions")
for op, v in ops.most_common(top):
    print(f"  {op:10s} {v / T * 100:5.1f}% inst  {stall[op] / S * 100:5.1f}% samples")
