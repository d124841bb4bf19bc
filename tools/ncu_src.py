"""Per-instruction stall breakdown of an ncu report: python tools/ncu_src.py REP [reason] [top] -- the
SASS listing with the sampled stall reasons, sorted by a reason (default all), and the samples summed
over address ranges (use to find which loop phase the time goes to)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
reason = sys.argv[2] if len(sys.argv) > 2 else "all"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
ia, isrc, iall, iex = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), \
    h.index("Instructions Executed")
data = []
for r in rows[2:]:
    if len(r) <= iall:
        continue
    st = {c: int(r[h.index(c)] or 0) for c in cols}
    data.append((int(r[iall] or 0), r[ia], r[isrc].strip(), st, int(r[iex] or 0)))
key = (lambda d: d[0]) if reason == "all" else (lambda d: d[3].get("stall_" + reason, 0))
if reason == "listing":
    for s, a, t, st, ex in data:
        big = ", ".join(f"{k[6:]}={v}" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:3] if v)
        print(f"{a[-5:]} {s:6d} ex={ex:9d} {t[:60]:60s} {big}")
    sys.exit()
for s, a, t, st, ex in sorted(data, key=key, reverse=True)[:top]:
    big = ", ".join(f"{k[6:]}={v}" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:4] if v)
    print(f"{s:6d} {a[-5:]} {t[:64]:64s} {big}")
