"""One GPU: the BASELINE.json configs c1-c4 (per-GPU shapes), stage split and total.
Usage: python tools/prof_configs.py [c1 c2 c3 c4]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2111_11148_b200 import _abi, dist  # noqa: E402
from paper_2111_11148_b200 import cholqr as cq  # noqa: E402

CONFIGS = {  # name: (method, m, n, kappa or sigma-rule, l)
    "c1": (_abi.RLU, 1_000_000, 128, 1e14, 256),
    "c2": (_abi.RQR_GAUSSIAN, 4_000_000, 256, 1e12, 512),
    "c3": (_abi.RQR_GAUSSIAN, 4_194_304, 64, 1e15, 128),
    "c4": (_abi.RLU, 1_000_000, 512, "two-segment", 768),
}


def sigma_c4(n):
    s = np.full(n, 1e-8)
    s[:256] = 10.0 ** (-8.0 * np.arange(256) / 255.0)
    return s


ctx = dist.make_context(0, 0, 1)
for name in (sys.argv[1:] or list(CONFIGS)):
    meth, m, n, kap, l = CONFIGS[name]
    sig = sigma_c4(n) if kap == "two-segment" else cq.geometric_sigma(n, kap)
    a = cq.synthesize_dev(m, n, sigma=sig, seed=1, ctx=ctx)
    cfg = cq.SketchConfig(strategy=cq.Strategy.Gaussian, size=l, seed=cq.derive(1, 0x5E7C))
    q = torch.empty_like(a)
    times, rep = [], None
    for it in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, r, rep = dist.factor_sharded(ctx, meth, a, m, 0, cfg, _abi.options(), q_out=q)
        torch.cuda.synchronize()
        if it:
            times.append(time.perf_counter() - t0)
    orth = cq.orthogonality_error_dev(q, ctx)
    flops = 2.0 * l * m * n + 2.0 * m * n * n + m * n * (n + 1)
    t = min(times)
    print(f"{name}: {_abi.METHOD_NAMES[meth]} m={m} n={n} l={l}: {t * 1e3:.2f} ms  {flops / t / 1e12:.1f} TFLOP/s  "
          f"orth {orth:.1e}  stages {[round(x, 2) for x in rep.stage_ms]}", flush=True)
    del a, q
    torch.cuda.empty_cache()
