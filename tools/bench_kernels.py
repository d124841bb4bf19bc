"""Per-stage device timings on the c1 shape (CUDA events via the report), for A/B runs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402  (workload tables)
from paper_2111_11148_b200 import _abi, dist  # noqa: E402
from paper_2111_11148_b200 import cholqr as cq  # noqa: E402

m = int(os.environ.get("PROF_M", 1_000_000))
n = int(os.environ.get("PROF_N", 128))
methods = os.environ.get("PROF_METHODS", "rlu").split(",")
dev = torch.device("cuda", 0)
ctx = dist.make_context(0, 0, 1)
kap = os.environ.get("PROF_KAPPA", "1e14")
a = cq.synthesize_dev(m, n, seed=1, sigma=bench.workload_sigma(n, kap if kap == "two-segment" else float(kap)), ctx=ctx)
cfg = cq.SketchConfig(strategy=cq.Strategy.Gaussian, rate=float(os.environ.get("PROF_RATE", "2.0")),
                      seed=cq.derive(1, 0x5E7C))
q = torch.empty_like(a)
ids = {"rlu": _abi.RLU, "rqr": _abi.RQR_GAUSSIAN, "cholqr2": _abi.CHOLQR2, "scholqr3": _abi.SCHOLQR3,
       "rqr-uniform": _abi.RQR, "cholqr": _abi.CHOLQR}
for name in methods:
    meth = ids[name]
    opts = _abi.options(shift_kind=_abi.SHIFT_FIXED, shift_value=1e-15)
    for _ in range(3):
        dist.factor_sharded(ctx, meth, a, m, 0, cfg, opts, q_out=q)
    tot = np.zeros(7)
    K = 5
    for _ in range(K):
        _, r, rep = dist.factor_sharded(ctx, meth, a, m, 0, cfg, opts, q_out=q)
        tot += np.array(rep.stage_ms[:])
    tot /= K
    print(f"{name:10s} m={m} n={n} total {tot.sum():8.3f} ms | " +
          " ".join(f"{k}={v:.3f}" for k, v in zip(_abi.STAGE_NAMES, tot) if v > 0),
          f"| orth={cq.orthogonality_error_dev(q, ctx):.2e}")
