"""Per-root time by level regime from a bench --dump-levels file (which kind of
level a change moved):  python tools/level_classes.py levels.json [levels2.json ...]"""
import json
import sys

for path in sys.argv[1:]:
    d = json.load(open(path))
    n = d["n_plus"]
    cls = {}
    nroots = len(d["roots"])
    for r in d["roots"]:
        reached = 1
        for i, l in enumerate(r["levels"]):
            U = n - reached
            nxt = r["levels"][i + 1]["n_f"] if i + 1 < len(r["levels"]) else 0
            t = l["seconds"] * 1e6
            if l["executed"] == "bottom_up":
                f = U / n
                key = ("BU U>1/2" if f > 0.5 else "BU 1/16<U<=1/2" if f > 1 / 16 else
                       "BU 1/256<U<=1/16" if f > 1 / 256 else "BU U<=1/256")
            else:
                key = "TD mf>=2^20" if l["m_f"] >= 1 << 20 else "TD mf<2^20"
            c = cls.setdefault(key, [0, 0.0])
            c[0] += 1
            c[1] += t
            reached += nxt
    print(path)
    for k, (c, t) in sorted(cls.items()):
        print(f"  {k:18s} levels {c:4d}  {t / nroots:7.1f} us/root  mean {t / c:6.1f} us")
    print(f"  total {sum(t for _, t in cls.values()) / nroots:.1f} us/root")
