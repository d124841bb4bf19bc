"""One c1 factorization (plus warm-up) for ncu launch lists / kernel captures."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2111_11148_b200 import _abi, dist  # noqa: E402
from paper_2111_11148_b200 import cholqr as cq  # noqa: E402

m = int(os.environ.get("PROF_M", bench.M_PER_GPU))
n = int(os.environ.get("PROF_N", bench.N))
method = {"rlu": _abi.RLU, "rqr": _abi.RQR_GAUSSIAN, "cholqr2": _abi.CHOLQR2}[os.environ.get("PROF_METHOD", "rlu")]
reps = int(os.environ.get("PROF_REPS", "2"))
dev = torch.device("cuda", 0)
ctx = dist.make_context(0, 0, 1)
a = bench.make_input(m, n, 0, 1, dev, ctx=ctx)
cfg = cq.SketchConfig(strategy=cq.Strategy.Gaussian, rate=2.0, seed=bench._seed_value())
q = torch.empty_like(a)
torch.cuda.synchronize()
torch.cuda.profiler.start()  # ncu --profile-from-start off: only the factorizations, not the input synthesis
for _ in range(reps):
    _, r, rep = dist.factor_sharded(ctx, method, a, m, 0, cfg, _abi.options(), q_out=q)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("stage_ms", [round(x, 3) for x in rep.stage_ms], "launches", ctx.launches)
