"""Per-call host overhead of cqr_factor_dev: c1 time per call vs the sum of its stage events, and a tiny
problem's per-call time (mostly host work and launch latency)."""
import ctypes as C
import sys
import time

sys.path.insert(0, "/root/repo")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2111_11148_b200 import _abi, dist  # noqa: E402
from paper_2111_11148_b200 import cholqr as cq  # noqa: E402

ctx = dist.make_context(0, 0, 1)
stream = torch.cuda.ExternalStream(ctx.stream, device="cuda:0")
for m in (2048, 1000000):
    n = 128
    a = cq.synthesize_dev(m, n, 1e14, 1, ctx=ctx)
    q = torch.empty_like(a)
    cfg = cq.SketchConfig(strategy=cq.Strategy.Gaussian, size=2 * n, seed=cq.derive(1, 0x5E7C))
    opts = _abi.options()
    for _ in range(5):
        dist.factor_sharded(ctx, _abi.RLU, a, m, 0, cfg, opts, q_out=q)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    K = 30
    st = np.zeros(_abi.STAGE_COUNT)
    t0 = time.perf_counter()
    e0.record(stream)
    for _ in range(K):
        _, _, rep = dist.factor_sharded(ctx, _abi.RLU, a, m, 0, cfg, opts, q_out=q)
        st += np.array(rep.stage_ms[:])
    e1.record(stream)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / K * 1e3
    ev = e0.elapsed_time(e1) / K
    # the raw C call, arguments prepared once
    cfg_c = cfg._c()
    r = np.zeros((n, n))
    rep = _abi.Report()
    lib = cq._lib()
    args = (ctx.h, _abi.RLU, C.c_void_p(a.data_ptr()), m, m, 0, n, a.stride(0), C.byref(cfg_c), C.byref(opts),
            C.c_void_p(q.data_ptr()), q.stride(0), cq._ptr(r), n, C.byref(rep))
    torch.cuda.synchronize()
    e0.record(stream)
    t0 = time.perf_counter()
    for _ in range(K):
        lib.cqr_factor_dev(*args)
    e1.record(stream)
    torch.cuda.synchronize()
    wall_raw = (time.perf_counter() - t0) / K * 1e3
    print(f"m={m}: events {ev:.3f} ms/call, wall {wall:.3f}, stage sum {st.sum() / K:.3f}, raw C call wall "
          f"{wall_raw:.3f} / events {e0.elapsed_time(e1) / K:.3f}, launches/call {ctx.launches}", flush=True)
