"""Per-kernel summary of an ncu metrics CSV (gpu__time_duration.sum, dram__bytes_read.sum,
dram__bytes_write.sum): time share per kernel and the dominant kernel's DRAM bytes per launch.
python tools/traffic_summary.py <csv> <workload> [--json profiles/traffic.json]"""
import csv
import json
import sys
from collections import defaultdict

path, workload = sys.argv[1], sys.argv[2]
rows = [r for r in csv.DictReader(l for l in open(path) if l.startswith('"'))]
by = defaultdict(lambda: {"launches": set(), "time_us": 0.0, "read": 0.0, "write": 0.0})
unit = {"ms": 1e3, "us": 1.0, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "nsecond": 1e-3}
bunit = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
for r in rows:
    k = r["Kernel Name"].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
    d = by[k]
    d["launches"].add(r["ID"])
    v = float(r["Metric Value"].replace(",", ""))
    name, u = r["Metric Name"], r["Metric Unit"]
    if name == "gpu__time_duration.sum":
        d["time_us"] += v * unit.get(u, 1.0)
    elif name == "dram__bytes_read.sum":
        d["read"] += v * bunit.get(u, 1.0)
    elif name == "dram__bytes_write.sum":
        d["write"] += v * bunit.get(u, 1.0)
tot = sum(d["time_us"] for d in by.values())
out = sorted(by.items(), key=lambda kv: -kv[1]["time_us"])
for k, d in out:
    nl = len(d["launches"])
    print(f"{d['time_us'] / tot * 100:5.1f}%  {d['time_us']:9.1f} us  x{nl:<3d} {(d['read'] + d['write']) / nl / 1e6:9.1f} MB/launch  {k[:90]}")
if "--json" in sys.argv:
    jp = sys.argv[sys.argv.index("--json") + 1]
    try:
        js = json.load(open(jp))
    except Exception:
        js = {}
    k, d = out[0]
    nl = len(d["launches"])
    js[workload] = {"kernel": k, "bytes_per_launch": (d["read"] + d["write"]) / nl, "read": d["read"] / nl,
                    "write": d["write"] / nl, "share": d["time_us"] / tot, "source": path}
    json.dump(js, open(jp, "w"), indent=1)
