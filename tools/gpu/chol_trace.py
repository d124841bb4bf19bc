"""clock64 marks of chol_reg_kernel (library built with -DCQR_LU_TRACE): per step, row lanes' shuffle ->
sqrt/rcp -> divisions+stores, and thread 0 past the barrier."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

from oracle import oracle as o  # noqa: E402
from paper_2111_11148_b200 import cholqr as cq  # noqa: E402

n = int(os.environ.get("PROF_N", 128))
g = o.gram(o.gaussian_matrix(4 * n, n, 3))
for _ in range(2):
    cq.cholesky_upper(g)
buf = np.zeros(1024, dtype=np.int64)
assert cq._lib().cqr_debug_lu_trace(C.c_void_p(buf.ctypes.data)) == 0
t = buf[500:756].reshape(64, 4)
for i in range(1, 20):
    print(f"step {i:3d}: s_bad read(i-1)->row start {t[i,0]-t[i-1,3]:6d}  sqrt+rcp+ok {t[i,1]-t[i,0]:6d}  div {t[i,2]-t[i,1]:6d}  "
          f"->STS+barrier+s_bad read {t[i,3]-t[i,2]:6d}  step total {t[i,3]-t[i-1,3]:6d}")
