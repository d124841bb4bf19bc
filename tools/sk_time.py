"""Time the device Gaussian sketch alone (cqr_sketch_gaussian_dev) at (m, n, l): CUDA events around
repeated calls (each call = pre-pass + sketch kernel + reduce + a sync)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2111_11148_b200 import cholqr as G  # noqa: E402

m, n, l = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
ctx = G.context(0)
a = torch.randn(m, n, dtype=torch.float64, device="cuda")
a1 = torch.empty(l, n, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()


def call():
    st = G._lib().cqr_sketch_gaussian_dev(ctx.h, C.c_void_p(a.data_ptr()), m, m, 0, n, n, l, 12345,
                                          C.c_void_p(a1.data_ptr()))
    assert st == 0, ctx.last_error()


for _ in range(3):
    call()
ts = []
for _ in range(7):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    call()
    e.record()
    torch.cuda.synchronize()
    ts.append(s.elapsed_time(e))
ms = sorted(ts)[3]
print(f"{os.environ.get('CQR_LIB', 'libcqr.so')}: sketch m={m} n={n} l={l}: {ms:.3f} ms "
      f"({2 * l * m * n / ms / 1e9:.1f} TFLOP/s)", flush=True)
