"""Recompute bench.py's roofline.by_direction from a --dump-levels file:
  python tools/roofline_from_levels.py profiles/r02_levels_s26.json
(sum of byte-model bytes / sum of level device time per executed direction,
over every timed root, against the peak the bench used)."""
import json
import sys

d = json.load(open(sys.argv[1]))
peak = d["peak_gbs"]
for kind in ("top_down", "bottom_up"):
    B = sum(lv["bytes"] for r in d["roots"] for lv in r["levels"] if lv["executed"] == kind)
    T = sum(lv["seconds"] for r in d["roots"] for lv in r["levels"] if lv["executed"] == kind)
    big = [max((lv for lv in r["levels"] if lv["executed"] == kind), key=lambda x: x["bytes"], default=None)
           for r in d["roots"]]
    big = [x for x in big if x]
    bb = sum(x["bytes"] for x in big) / sum(x["seconds"] for x in big) / 1e9 if big else 0.0
    print(f"{kind:9s}: {B / 1e9:8.3f} GB in {T * 1e3:8.3f} ms -> {B / T / 1e9:7.1f} GB/s = {B / T / 1e9 / peak:.3f} "
          f"of {peak:.0f} GB/s; largest level per root {bb:7.1f} GB/s = {bb / peak:.3f}")
tot_b = sum(lv["bytes"] for r in d["roots"] for lv in r["levels"])
tot_t = sum(r["mean_s"] for r in d["roots"])
print(f"whole kernel: {tot_b / tot_t / 1e9:.1f} GB/s = {tot_b / tot_t / 1e9 / peak:.3f} (bytes / mean launch time)")
