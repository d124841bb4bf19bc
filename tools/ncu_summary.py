"""Summarise ncu launch lists / --set full reports into profiles/ (run here, no GPU)."""
import csv
import io
import subprocess
import sys
from collections import OrderedDict


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    out = []
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1.0)
        out.append((r[ki], v))
    return out


def details(rep, names=("Duration", "DRAM Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
                        "Achieved Occupancy", "Registers Per Thread", "Dynamic Shared Memory Per Block",
                        "L1/TEX Hit Rate", "L2 Hit Rate", "Issue Slots Busy")):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h = rows[0]
    res = OrderedDict()
    for r in rows[1:]:
        d = dict(zip(h, r))
        k = d.get("Kernel Name", "")[:60] + " #" + d.get("ID", "")
        if d.get("Metric Name") in names:
            res.setdefault(k, OrderedDict())[d["Metric Name"]] = d["Metric Value"] + " " + d["Metric Unit"]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    if rr:
        h = rr[0]
        want = ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed_pipe_fp64.sum",
                "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "gpu__time_duration.sum",
                "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]
        idx = {w: h.index(w) for w in want if w in h}
        for r in rr[2:]:
            k = r[h.index("Kernel Name")][:60] + " #" + r[h.index("ID")]
            for w, i in idx.items():
                res.setdefault(k, OrderedDict())[w] = r[i] + " " + rr[1][i]
    return res


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        tot = 0.0
        for name, us in launches(sys.argv[2]):
            if "cqr" in name or "unnamed>::" in name or "finite" in name:
                print(f"{us:10.1f} us  {name[:110]}")
                tot += us
        print(f"{tot:10.1f} us  total (cqr kernels)")
    else:
        for k, v in details(sys.argv[2]).items():
            print(k)
            for a, b in v.items():
                print(f"    {a:70s} {b}")
