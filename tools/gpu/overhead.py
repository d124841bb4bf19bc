import sys, time
sys.path.insert(0, '/root/repo')
import torch
from paper_2111_11148_b200 import _abi, dist
from paper_2111_11148_b200 import cholqr as cq
ctx = dist.make_context(0, 0, 1)
for m in (2048, 1000000):
    a = cq.synthesize_dev(m, 128, 1e6, 1, ctx=ctx)
    q = torch.empty_like(a)
    cfg = cq.SketchConfig(strategy=cq.Strategy.Gaussian, seed=3)
    for _ in range(5): dist.factor_sharded(ctx, _abi.RLU, a, m, 0, cfg, q_out=q)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(50): dist.factor_sharded(ctx, _abi.RLU, a, m, 0, cfg, q_out=q)
    torch.cuda.synchronize()
    print(m, "ms/factorization", (time.perf_counter() - t0) / 50 * 1e3)
