"""Aggregate ncu source-page metrics by CUDA source line.

  ncu -i rep.ncu-rep --page source --csv --print-source cuda,sass > src.csv
  python tools/ncu_lines.py src.csv [top] [column]

column defaults to "Warp Stall Sampling (All Samples)"; e.g. "Instructions Executed".
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
col = sys.argv[3] if len(sys.argv) > 3 else "Warp Stall Sampling (All Samples)"
hdr = None
func = None
acc = {}
for r in rows:
    if r and r[0] == "Function Name":
        func = r[1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0].isdigit():
        i = hdr.index(col)
        try:
            s = int(float(r[i].replace(",", "")))
        except ValueError:
            continue
        key = (func[:40], int(r[0]), r[1].strip()[:80])
        acc[key] = acc.get(key, 0) + s
tot = sum(acc.values()) or 1
print("total", col, tot)
for (f, ln, src), s in sorted(acc.items(), key=lambda x: -x[1])[:top]:
    print(f"{s:10d} {100 * s / tot:5.1f}%  L{ln:4d}  {src}")
