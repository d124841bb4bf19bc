"""CQR_TRACE=1 python tools/gpu/trace_call.py: the host/device timeline of c1 factorizations."""
import sys
sys.path.insert(0, "/root/repo")
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2111_11148_b200 import _abi, dist  # noqa: E402
from paper_2111_11148_b200 import cholqr as cq  # noqa: E402
ctx = dist.make_context(0, 0, 1)
m, n = 1_000_000, 128
a = cq.synthesize_dev(m, n, seed=bench.SEED, sigma=bench.workload_sigma(n, 1e14), ctx=ctx)
q = torch.empty_like(a)
cfg = cq.SketchConfig(strategy=cq.Strategy.Gaussian, size=256, seed=cq.derive(bench.SEED, 0x5E7C))
for _ in range(8):
    dist.factor_sharded(ctx, _abi.RLU, a, m, 0, cfg, _abi.options(), q_out=q)
torch.cuda.synchronize()
