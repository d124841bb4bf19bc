import os, sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from oracle import oracle as o
from paper_2111_11148_b200 import _abi, cholqr as G
o.set_test_threads(os.cpu_count())
for kappa in (1e9, 1e10, 1e11):
    a = G.synthesize_dev(100000, 100, kappa, 3)
    ah = np.ascontiguousarray(a.cpu().numpy())
    sv = np.linalg.svd(ah, compute_uv=False)
    cfg = G.SketchConfig(rate=2.0, seed=G.derive(3, 0x5E7C))
    for meth in (_abi.RQR, _abi.RLU):
        f, _, rep = G._factor(meth, ah, cfg, _abi.options(diagnostics=True))
        ref = o.factor(meth, ah, cfg._c(), _abi.options(diagnostics=True), workers=16)
        print(kappa, _abi.METHOD_NAMES[meth], "sv", sv[0], sv[-1], "retries", f.report.stages[0].retries, ref.stages[0].retries,
              "cond_x gpu", f.report.stages[1].cond_x, "orc", ref.stages[1].cond_x,
              "orth gpu", o.orthogonality_error(f.q), "orc", o.orthogonality_error(ref.q),
              "dR", np.linalg.norm(f.r - ref.r) / np.linalg.norm(ref.r), flush=True)
    # the sketch: uniform rows, and R~ of the device QR kernel vs the oracle's
    sk = G.sample_rows_uniform(ah, cfg)
    print(" idx unique", len(set(sk.indices.tolist())), "of", len(sk.indices))
    rt = G.qr_r_factor(sk.a1); rto = o.qr_r_factor(sk.a1) if hasattr(o, 'qr_r_factor') else None
    if rto is not None:
        print(" R~ rel diff", np.linalg.norm(rt - rto) / np.linalg.norm(rto), "cond R~", np.linalg.cond(rto))
