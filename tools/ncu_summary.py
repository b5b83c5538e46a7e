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
    """Per kernel: launches, device time (ms) and -- when captured -- DRAM bytes
    read + written and the resulting GB/s."""
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
    h = rows[0]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    ii = h.index("ID") if "ID" in h else None
    tscale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
    bscale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    agg = {}
    for r in rows[1:]:
        name = r[ki].split("(")[0][:72]
        a = agg.setdefault(name, {"ms": 0.0, "bytes": 0.0, "ids": set()})
        v = float(r[vi].replace(",", ""))
        if r[mi] == "gpu__time_duration.sum":
            a["ms"] += v * tscale.get(r[ui], 1e-6)
            a["ids"].add(r[ii] if ii is not None else len(a["ids"]))
        elif r[mi].startswith("dram__bytes"):
            a["bytes"] += v * bscale.get(r[ui], 1.0)
    tot = sum(a["ms"] for a in agg.values())
    print(f"# {title}")
    print("# ncu --metrics gpu__time_duration.sum[,dram__bytes_read.sum,dram__bytes_write.sum] --clock-control none")
    print("# (cold-cache, serialised replays: compare shares, not absolute times)")
    print(f"# total device time {tot:.3f} ms over {sum(len(a['ids']) for a in agg.values())} launches")
    print("share%   total_ms    n   DRAM_GB   GB/s   kernel")
    for name, a in sorted(agg.items(), key=lambda x: -x[1]["ms"]):
        gbs = a["bytes"] / (a["ms"] * 1e-3) / 1e9 if a["ms"] > 0 and a["bytes"] > 0 else 0.0
        print(f"{100 * a['ms'] / tot:6.2f} {a['ms']:10.3f} {len(a['ids']):4d} {a['bytes'] / 1e9:9.3f} {gbs:7.0f}   {name}")


def full(rep, command, name=None):
    """Key metrics per launch of a --set full capture (a .ncu-rep, or its
    `--page raw --csv` export as .csv / .csv.gz)."""
    if rep.endswith(".csv.gz"):
        import gzip

        out = gzip.open(rep, "rt").read()
    elif rep.endswith(".csv"):
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = {"command": command, "units": {k: units[h.index(k)] for k in KEYS if k in h}, "launches": []}
    scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "Tbyte": 1e6}
    for r in rows[2:]:
        d = {k: r[h.index(k)] for k in KEYS if k in h}
        mb = 0.0  # DRAM traffic of the launch in MB (units differ per metric and per report)
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            if k in h:
                mb += float(r[h.index(k)].replace(",", "")) * scale.get(units[h.index(k)], 1.0)
        d["dram_MB"] = round(mb, 3)
        t = float(d.get("gpu__time_duration.sum", "0").replace(",", "")) if "gpu__time_duration.sum" in d else 0.0
        tu = units[h.index("gpu__time_duration.sum")] if "gpu__time_duration.sum" in h else "us"
        t_us = t * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(tu, 1.0)
        d["dram_TBps"] = round(mb / t_us, 3) if t_us > 0 else None
        if "lts__t_sectors.sum" in h:
            d["lts__t_sectors.sum"] = r[h.index("lts__t_sectors.sum")]
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
