"""Per-source-line stall breakdown of an ncu report (--import-source on), per kernel.
Usage: python tools/ncu_lines.py <rep> [top] [kernel-substring]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
want = sys.argv[3] if len(sys.argv) > 3 else ""
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
hdr = None
fname = func = ""
per = {}
for r in csv.reader(io.StringIO(src)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        func = r[1].split("(")[0]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0] != "":  # headers differ per file section: key each row by its own
        per.setdefault(func, []).append((fname, {**dict(zip(hdr, r)), "Source": r[1]}))


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


reasons = sorted({h for rows in per.values() for _, r in rows for h in r
                  if h.startswith("stall_") and "Not Issued" not in h})
idx = {k: k for k in reasons}
tot_i = "Warp Stall Sampling (All Samples)"
ins_i = "Instructions Executed"
for func, rows in per.items():
    if want not in func:
        continue
    T = sum(f(r[tot_i]) for _, r in rows) or 1
    agg = {k: sum(f(r.get(idx[k], '0')) for _, r in rows) / T * 100 for k in reasons}
    print(f"== {func}  (samples {int(T)})")
    print("overall:", ", ".join(f"{k[6:]} {v:.1f}%" for k, v in sorted(agg.items(), key=lambda kv: -kv[1]) if v > 0.5))
    for fn, r in sorted(rows, key=lambda x: -f(x[1][tot_i]))[:top]:
        parts = sorted(((f(r.get(idx[k], '0')), k[6:]) for k in reasons), reverse=True)[:3]
        print(f"{f(r[tot_i]) / T * 100:5.1f}% {fn}:{r["Line No"]:>4} inst={int(f(r[ins_i])):>10} "
              + " ".join(f"{n}={v / max(f(r[tot_i]), 1) * 100:.0f}%" for v, n in parts if v > 0) + f" | {r["Source"].strip()[:70]}")
