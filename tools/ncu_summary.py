"""Summaries of ncu output for profiles/.

  python tools/ncu_summary.py launches <launches.csv> <title>      # launch list -> share table
  python tools/ncu_summary.py full <rep.ncu-rep> <command> [name] # key metrics of one --set full capture (JSON)
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
]
STALLS = "smsp__pcsamp_warps_issue_stalled_"


def launches(path, title):
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = {}
    for r in rows[1:]:
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(r[ui], 1e-6)
        name = r[ki].split("(")[0][:72]
        t, c = agg.get(name, (0.0, 0))
        agg[name] = (t + float(r[vi].replace(",", "")) * scale, c + 1)
    tot = sum(t for t, _ in agg.values())
    print(f"# {title}")
    print("# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised: compare shares)")
    print(f"# total device time {tot:.3f} ms over {sum(c for _, c in agg.values())} launches")
    print("share%   total_ms  n     kernel")
    for name, (t, c) in sorted(agg.items(), key=lambda x: -x[1][0]):
        print(f"{100 * t / tot:6.2f} {t:10.3f} {c:4d}  {name}")


def full(rep, command, name=None):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = {"command": command, "units": {k: units[h.index(k)] for k in KEYS if k in h}, "launches": []}
    for r in rows[2:]:
        d = {k: r[h.index(k)] for k in KEYS if k in h}
        st = {k[len(STALLS):]: float(r[i].replace(",", "")) for i, k in enumerate(h)
              if k.startswith(STALLS) and not k.endswith("not_issued") and r[i].replace(",", "").replace(".", "").isdigit()}
        tot = sum(st.values()) or 1.0
        d["stall_share_top"] = {k: round(v / tot, 3) for k, v in sorted(st.items(), key=lambda x: -x[1])[:6]}
        res["launches"].append(d)
    if name:
        res["workload"] = name
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
