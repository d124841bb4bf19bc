"""Per-warp step timeline of sketch_ws_kernel CTA 0 (library built with -DCQR_WS_TRACE)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2111_11148_b200 import cholqr as cq  # noqa: E402

m, n = 1_000_000, int(os.environ.get("PROF_N", 128))
l = 2 * n
a = torch.randn(m, n, dtype=torch.float64, device="cuda")
a1 = torch.empty(l, n, dtype=torch.float64, device="cuda")
ctx = cq.context(0)
lib = cq._lib()
for _ in range(2):
    ctx._check(lib.cqr_sketch_gaussian_dev(ctx.h, C.c_void_p(a.data_ptr()), m, m, 0, n, n, l, 12345,
                                           C.c_void_p(a1.data_ptr())))
torch.cuda.synchronize()
buf = np.zeros(16 * 64 * 2, dtype=np.int64)
assert lib.cqr_debug_trace(C.c_void_p(buf.ctypes.data)) == 0
t = buf.reshape(16, 64, 2)
t0 = t[:, 16, 0].min()
print("step | MMA start..end (min/max over 8 warps)      | GEN start..done (min/max over 8 warps)")
for s in range(16, 40):
    ms, me, gs, gd = t[:8, s, 0] - t0, t[:8, s, 1] - t0, t[8:, s, 0] - t0, t[8:, s, 1] - t0
    print(f"{s:4d} | {ms.min():7d}-{ms.max():7d} .. {me.min():7d}-{me.max():7d} | "
          f"{gs.min():7d}-{gs.max():7d} .. {gd.min():7d}-{gd.max():7d}")
mma = (t[:8, 17:63, 1] - t[:8, 17:63, 0]).mean()
step = (t[:8, 62, 0] - t[:8, 17, 0]).mean() / 45
gen = (t[8:, 17:63, 1] - t[8:, 17:63, 0]).mean()
print(f"avg step {step:.0f} clk, MMA busy {mma:.0f} clk/step, GEN busy {gen:.0f} clk/step")
