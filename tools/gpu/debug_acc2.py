import os, sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from oracle import oracle as o
from paper_2111_11148_b200 import _abi, cholqr as G
o.set_test_threads(os.cpu_count())
FIXED = G.ShiftMode.fixed(1e-15)
seeds = [int(x) for x in sys.argv[1:]] or [1, 2, 3]
if os.environ.get("PRE"):
    for meth, m, n, l in ((_abi.RLU, 200000, 128, 256), (_abi.RQR_GAUSSIAN, 100000, 256, 512), (_abi.RQR_GAUSSIAN, 262144, 64, 128), (_abi.RLU, 60000, 512, 768)):
        if os.environ["PRE"] != "all" and str(n) not in os.environ["PRE"].split(","):
            continue
        a = G.synthesize_dev(m, n, 1e8, 1)
        ah = np.ascontiguousarray(a.cpu().numpy())
        cfg = G.SketchConfig(strategy=G.Strategy.Gaussian, size=l, seed=5)
        G._factor(meth, ah, cfg, _abi.options())
        print("pre", n, flush=True)
for seed in seeds:
    for e in range(3, 16):
        kappa = 10.0 ** e
        a = G.synthesize_dev(100000, 100, kappa, seed)
        for method in (_abi.RQR, _abi.RLU, _abi.SCHOLQR3):
            cfg = G.SketchConfig(rate=2.0, seed=G.derive(seed, 0x5E7C))
            opts = G._opts(G.Options(), FIXED)
            f, _, rep = G._factor(method, a, cfg, opts)
            orth = G.orthogonality_error_dev(f.q)
            if os.environ.get("RES"):
                G.residual_error_dev(a, f.q, f.r)
            if orth > 1e-11:
                ah = np.ascontiguousarray(a.cpu().numpy())
                qh = f.q.cpu().numpy()
                fh, _, reph = G._factor(method, ah, cfg, opts)
                ref = o.factor(method, ah, cfg._c(), opts, workers=16)
                f2, _, _ = G._factor(method, a, cfg, opts)
                print("FAIL", seed, kappa, _abi.METHOD_NAMES[method], "orth dev", orth, "orth(q) by oracle", o.orthogonality_error(qh),
                      "host-path orth", o.orthogonality_error(fh.q), "oracle", o.orthogonality_error(ref.q),
                      "rerun orth", G.orthogonality_error_dev(f2.q), "same q rerun", torch.equal(f.q, f2.q),
                      "dq host", np.abs(qh - fh.q).max(), "retries", rep.stages[0].retries, reph.stages[0].retries,
                      "dR", np.abs(f.r - fh.r).max(), flush=True)
                bad = np.argwhere(np.abs(qh - fh.q) > 1e-8)
                qs = [G._factor(method, a, cfg, opts)[0].q for _ in range(6)]
                print("  reruns equal to first:", [torch.equal(qs[0], x) for x in qs], "orths", [G.orthogonality_error_dev(x) for x in qs], flush=True)
                print("  bad rows", np.unique(bad[:, 0])[:20], len(np.unique(bad[:, 0])), "cols", np.unique(bad[:, 1])[:20], flush=True)
print("done")
