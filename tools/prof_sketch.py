"""Gaussian sketch only (cqr_sketch_gaussian_dev), c1 shape, CUDA-event timed."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2111_11148_b200 import cholqr as cq  # noqa: E402

m = int(os.environ.get("PROF_M", 1_000_000))
n = int(os.environ.get("PROF_N", 128))
l = int(os.environ.get("PROF_L", 2 * n))
a = torch.randn(m, n, dtype=torch.float64, device="cuda")
a1 = torch.empty(l, n, dtype=torch.float64, device="cuda")
ctx = cq.context(0)
lib = cq._lib()


def run():
    ctx._check(lib.cqr_sketch_gaussian_dev(ctx.h, C.c_void_p(a.data_ptr()), m, m, 0, n, n, l, 12345,
                                           C.c_void_p(a1.data_ptr())))


for _ in range(int(os.environ.get("PROF_REPS", "3"))):
    run()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(5):
    run()
e.record()
torch.cuda.synchronize()
t = s.elapsed_time(e) / 5
print(f"sketch m={m} n={n} l={l}: {t:.3f} ms per call ({2 * l * m * n / t / 1e9:.1f} TFLOP/s)")
