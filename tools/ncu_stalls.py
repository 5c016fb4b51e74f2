"""Stall reasons by source line (and totals) from an ncu 'cuda,sass' source
page CSV: ncu -i rep --page source --csv --print-source cuda,sass > x.csv
python tools/ncu_stalls.py x.csv [file:line-lo-hi ...]   (ranges optional)"""
import csv, sys, re
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
ranges = []
for a in sys.argv[2:]:
    m = re.match(r"(.+):(\d+)-(\d+)", a)
    ranges.append((m.group(1), int(m.group(2)), int(m.group(3))))
agg = defaultdict(lambda: defaultdict(float))
tot = defaultdict(float)
cur_file, header, cur_line = "?", None, None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        header = {name: i for i, name in enumerate(r)}
        reasons = [n for n in header if n.startswith("stall_") and "Not Issued" not in n]
        continue
    if header is None or r[0] == "Function Name":
        continue
    if r[0]:
        cur_line = int(r[0])
        continue
    if r[2] in ("...", "-"):
        continue
    for n in reasons:
        try:
            v = float(r[header[n]] or 0)
        except ValueError:
            v = 0.0
        agg[(cur_file, cur_line)][n] += v
        tot[n] += v
T = sum(tot.values())
print("all:", " ".join(f"{k[6:]}={v / T * 100:.1f}%" for k, v in sorted(tot.items(), key=lambda kv: -kv[1]) if v))
for f, lo, hi in ranges:
    sub = defaultdict(float)
    for (ff, ln), d in agg.items():
        if ff == f and lo <= ln <= hi:
            for k, v in d.items():
                sub[k] += v
    S = sum(sub.values())
    print(f"{f}:{lo}-{hi}: {S / T * 100:.1f}% of samples:",
          " ".join(f"{k[6:]}={v / max(S, 1) * 100:.0f}%" for k, v in sorted(sub.items(), key=lambda kv: -kv[1]) if v))
