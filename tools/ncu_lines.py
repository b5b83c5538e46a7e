"""Aggregate ncu warp-stall samples by CUDA source line.

  ncu -i rep.ncu-rep --page source --csv --print-source cuda,sass > src.csv
  python tools/ncu_lines.py src.csv [top]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
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
        i = hdr.index("Warp Stall Sampling (All Samples)")
        try:
            s = int(r[i])
        except ValueError:
            continue
        key = (func[:40], int(r[0]), r[1].strip()[:80])
        acc[key] = acc.get(key, 0) + s
tot = sum(acc.values()) or 1
print("total samples", tot)
for (f, ln, src), s in sorted(acc.items(), key=lambda x: -x[1])[:top]:
    print(f"{s:7d} {100 * s / tot:5.1f}%  L{ln:4d}  {src}")
