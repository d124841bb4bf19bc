"""One factorization of a BASELINE.json workload (after warm-up) between cudaProfilerStart/Stop, for ncu
launch lists and metric captures: python tools/prof_one.py [c1|c2|c3|c4]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2111_11148_b200 import _abi, dist  # noqa: E402
from paper_2111_11148_b200 import cholqr as cq  # noqa: E402

w = sys.argv[1] if len(sys.argv) > 1 else "c1"
reps = int(os.environ.get("PROF_REPS", "1"))
mname, m_global, row0, m, n, l, kap, _, _ = bench.workload_shape(w, 1, 0)
method = {v: k for k, v in _abi.METHOD_NAMES.items()}[mname]
ctx = dist.make_context(0, 0, 1)
a = cq.synthesize_dev(m, n, seed=bench.SEED, sigma=bench.workload_sigma(n, kap), ctx=ctx)
cfg = cq.SketchConfig(strategy=cq.Strategy.Gaussian, size=l, seed=cq.derive(bench.SEED, 0x5E7C))
q = torch.empty_like(a)
for _ in range(2):
    dist.factor_sharded(ctx, method, a, m, 0, cfg, _abi.options(), q_out=q)
torch.cuda.synchronize()
torch.cuda.profiler.start()  # ncu --profile-from-start off: only these factorizations
for _ in range(reps):
    _, r, rep = dist.factor_sharded(ctx, method, a, m, 0, cfg, _abi.options(), q_out=q)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(w, "stage_ms", [round(x, 3) for x in rep.stage_ms], "launches", ctx.launches)
