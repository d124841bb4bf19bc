"""Phase marks of lu_rot_kernel (library built with -DCQR_LU_TRACE), c1 shape l=256 n=128."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

from paper_2111_11148_b200 import cholqr as cq  # noqa: E402

l, n = int(os.environ.get("PROF_L", 256)), int(os.environ.get("PROF_N", 128))
a = np.random.default_rng(1).standard_normal((l, n))
for _ in range(2):
    cq.lu_u_factor(a)
buf = np.zeros(1024, dtype=np.int64)
assert cq._lib().cqr_debug_lu_trace(C.c_void_p(buf.ctypes.data)) == 0
t0 = buf[0]
PW = int(os.environ.get("PROF_PW", 16))
for p in range((n + PW - 1) // PW):
    b = buf[1 + 4 * p: 5 + 4 * p] - t0
    print(f"panel {p}: start {b[0]:8d}  steps done {b[1]:8d} (+{b[1]-b[0]})  U12 done {b[3]:8d} (+{b[3]-b[1]})  "
          f"DMMA done {b[2 + 4 - 4 + 0] if False else buf[3 + 4 * p] - t0:8d}")
st = np.diff(buf[100:100 + n])
print("cycles per pivot step (panel 0):", st[:PW - 1].tolist())
print("mean per step, per panel:", [int(st[PW * p: PW * p + PW - 1].mean()) for p in range(n // PW)])
sub = buf[300:300 + 8 * 32].reshape(32, 8)
for j in range(1, 6):
    r = sub[j]
    print(f"step {j}: warp argmax+publish {r[0] - buf[100 + j]:5d} barrier {r[1] - r[0]:5d} "
          f"cross-warp {r[2] - r[1]:5d} update {r[3] - r[2]:5d} shift->next {buf[101 + j] - r[3]:5d}")
