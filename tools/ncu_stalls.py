"""Summarise an ncu report: key metrics + per-instruction stall samples (top N) + by opcode."""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, v = rows[0], rows[2]
keys = ["gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]
for k, x in zip(h, v):
    if k in keys or (k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")):
        if not k.startswith("smsp__pcsamp") or float(x or 0) > 0:
            print(f"{k:70s} {x}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hh = rows[1]
ia, isrc, iss = hh.index("Address"), hh.index("Source"), hh.index("Warp Stall Sampling (All Samples)")
data = [(int(r[iss] or 0), r[ia], r[isrc].strip()) for r in rows[2:] if len(r) > iss]
print("total samples", sum(d[0] for d in data))
for s, a, t in sorted(data, reverse=True)[:top]:
    print(f"{s:6d} {a[-5:]} {t[:100]}")
c = Counter()
for s, a, t in data:
    parts = t.split()
    if not parts:
        continue
    op = parts[1] if parts[0].startswith("@") else parts[0]
    c[op.split(".")[0]] += s
print(c.most_common(25))
