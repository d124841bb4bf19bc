"""Gram only, on the c1 shape (for timing / ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2111_11148_b200 import cholqr as cq  # noqa: E402

m = int(os.environ.get("PROF_M", 1_000_000))
n = int(os.environ.get("PROF_N", 128))
x = torch.randn(m, n, dtype=torch.float64, device="cuda")
for _ in range(int(os.environ.get("PROF_REPS", "3"))):
    g = cq.gram(x)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(5):
    g = cq.gram(x)
e.record()
torch.cuda.synchronize()
print(f"gram m={m} n={n}: {s.elapsed_time(e) / 5:.3f} ms per call (incl. combine + D2H)")
