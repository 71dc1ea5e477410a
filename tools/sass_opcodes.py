"""Static SASS opcode summary of the hot kernels in the built library
(cuobjdump -sass): per kernel the instruction count, the tensor-core / async-
copy / shuffle / atomic opcodes and the top opcodes.  Usage:
python tools/sass_opcodes.py [lib.so] > profiles/r2_sass_opcodes.md"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2510_12174_b200/libmsplat_b200.so"
HOT = ["forward_kernelIfLb1", "forward_pairs_kernelILi7", "backward_kernel_tcILb1", "backward_pairs_kernel",
       "preprocess_kernelIf", "projection_backward_kernelIf", "tile_sort_small_kernel", "tile_scatter_kernelILb1",
       "tile_hist_kernelILb1"]
KEY = ["HMMA", "LDGSTS", "UBLKCP", "UTMALDG", "UTCHMMA", "UTCQMMA", "SHFL", "RED", "ATOM", "ATOMS", "LDS", "STS",
       "LDG", "STG", "BAR", "VOTE", "MATCH", "DFMA", "DMUL", "FFMA", "MUFU"]
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs, cur = {}, None
for line in out.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        cur = m.group(1)
        funcs[cur] = collections.Counter()
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
    if m and cur:
        funcs[cur][m.group(1)] += 1
print("# SASS opcode summary (static, cuobjdump -sass of the in-tree libmsplat_b200.so, sm_100a)\n")
print("Static instruction counts per kernel (not executed counts).  `HMMA` = mma.sync TF32 (legacy warp MMA);")
print("`LDGSTS` = cp.async; `UBLKCP` / `UTMALDG` = TMA bulk / tensor copies; `UTC*MMA` = tcgen05.mma.\n")
print("| kernel | instructions | " + " | ".join(KEY) + " |")
print("|---|---|" + "---|" * len(KEY))
for h in HOT:
    names = [f for f in funcs if h in f]
    if not names:
        continue
    c = funcs[names[0]]
    print(f"| {h} | {sum(c.values())} | " + " | ".join(str(c.get(k, 0)) for k in KEY) + " |")
print()
for h in HOT:
    names = [f for f in funcs if h in f]
    if not names:
        continue
    c = funcs[names[0]]
    print(f"- **{h}** top opcodes: " + ", ".join(f"{k} {v}" for k, v in c.most_common(12)))
