"""Summarise an `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv` launch list into a markdown table (per kernel:
launches, device time, share, DRAM bytes) for the LAST fwd_bwd iteration, and
write per-launch DRAM traffic of the blend kernels to profiles/ncu_traffic.json.
Usage: python tools/summarize_launches.py <launches.csv> <out.md> [title]"""
import collections
import csv
import json
import os
import sys

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
ki, mi, vi, ui, idi = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
per = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    per.setdefault((int(r[idi]), r[ki]), {})[r[mi]] = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
ids = list(per.keys())
starts = [i for i, (_, k) in enumerate(ids) if "preprocess_kernel" in k]
seg = ids[starts[-1]:] if starts else ids
agg = collections.OrderedDict()
for key in seg:
    name = key[1].split("(")[0].replace("void ", "").replace("msplat_cuda::", "").replace("<unnamed>::", "")
    m = per[key]
    a = agg.setdefault(name, [0, 0.0, 0.0])
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0.0)
    a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
tot = sum(v[1] for v in agg.values())
title = sys.argv[3] if len(sys.argv) > 3 else "launch list"
out = [f"# {title}", "", "ncu `--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
       "--clock-control none`; last fwd_bwd iteration. Cold-cache and serialised: compare SHARES.", "",
       "| kernel | launches | device us | share | DRAM r+w per launch |", "|---|---|---|---|---|"]
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    out.append(f"| {k} | {v[0]} | {v[1]:.1f} | {v[1] / tot * 100:.1f}% | {v[2] / v[0] / 1e6:.1f} MB |")
out.append(f"| **total** | {sum(v[0] for v in agg.values())} | {tot:.1f} | 100% | "
           f"{sum(v[2] for v in agg.values()) / 1e6:.1f} MB (all) |")
open(sys.argv[2], "w").write("\n".join(out) + "\n")
print("\n".join(out))
# per-launch DRAM traffic of each timed stage (a stage may be several kernels:
# K9 = tensor-core phase A + pair-record phase B)
traffic = {}
for k, v in agg.items():
    for stage, prefs in (("backward", ("backward_kernel", "backward_pairs_kernel", "order_hist_kernel", "order_scatter_kernel")), ("forward", ("forward_kernel", "forward_pairs_kernel")),
                         ("preprocess", ("preprocess_kernel",)), ("proj_bwd", ("projection_backward_kernel",))):
        if any(k.startswith(pref) for pref in prefs):
            traffic[stage] = traffic.get(stage, 0.0) + v[2] / v[0]
# keyed by BASELINE config (bench.py reads its own config's entry; default cfg3)
cfg = sys.argv[4] if len(sys.argv) > 4 else "cfg3"
path = os.path.join(os.path.dirname(sys.argv[2]), "ncu_traffic.json")
try:
    allt = json.load(open(path))
    if not all(isinstance(v, dict) for v in allt.values()):
        allt = {}
except Exception:
    allt = {}
allt[cfg] = traffic
json.dump(allt, open(path, "w"), indent=1)
