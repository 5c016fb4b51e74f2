"""Aggregate an ncu 'cuda,sass' source-page CSV by source line.

usage: ncu -i rep --page source --csv --print-source cuda,sass > x.csv
       python tools/ncu_lines.py x.csv [top]
Prints per (file, line): stall samples, warp instructions executed,
thread instructions executed (SIMT efficiency) sorted by samples.
"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
agg = defaultdict(lambda: [0, 0, 0, ""])
cur_file, header, cur_line, cur_src = "?", None, None, ""
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        header = {name: i for i, name in enumerate(r)}
        continue
    if header is None or r[0] == "Function Name":
        continue
    if r[0]:
        cur_line, cur_src = r[0], r[1]
        continue
    if r[2] in ("...", "-"):
        continue
    def val(name):
        i = header.get(name)
        try:
            return float(r[i]) if i is not None and r[i] not in ("", "-") else 0.0
        except ValueError:
            return 0.0
    key = (cur_file, int(cur_line))
    a = agg[key]
    a[0] += val("Warp Stall Sampling (All Samples)")
    a[1] += val("Instructions Executed")
    a[2] += val("Thread Instructions Executed")
    a[3] = cur_src
tot = [sum(v[i] for v in agg.values()) for i in range(3)]
print(f"total samples {tot[0]:.0f}  warp insts {tot[1]:.3g}  SIMT {tot[2] / max(tot[1], 1) / 32:.2f}")
for (f, ln), (s, wi, ti, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{s / tot[0] * 100:5.1f}% {wi / tot[1] * 100:5.1f}%i simt={ti / max(wi, 1) / 32:.2f} "
          f"{f}:{ln:<4d} {src.strip()[:90]}")
