"""Time cqr_cholesky_upper's kernel alone (n x n, device-resident G) with CUDA events around repeated host calls
is too noisy; instead time the host call median over 50 runs (includes H2D/D2H of n^2 doubles)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from oracle import oracle as o  # noqa: E402
from paper_2111_11148_b200 import cholqr as cq  # noqa: E402
n = int(os.environ.get("PROF_N", 128))
g = o.gram(o.gaussian_matrix(4 * n, n, 3))
ts = []
for _ in range(60):
    t = time.perf_counter()
    try:
        cq.cholesky_upper(g)
    except Exception:
        pass
    ts.append(time.perf_counter() - t)
ts = sorted(ts[10:])
print(os.environ.get("CQR_LIB", "default"), f"n={n}: median host call {1e6 * ts[len(ts) // 2]:.1f} us")
