"""c4 at full size (1e6 x 512, l = 768, two-segment sigma): orthogonality and
residual of the B200 path next to the oracle's on the same A bytes and the same
Omega (the bench's c4 orth 2.46e-11 against the oracle's)."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from oracle import oracle as o  # noqa: E402
from paper_2111_11148_b200 import _abi  # noqa: E402
from paper_2111_11148_b200 import cholqr as G  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
n, l = 512, 768
sig = np.full(n, 1e-8)
sig[:256] = 10.0 ** (-8.0 * np.arange(256) / 255.0)
a = G.synthesize_dev(m, n, seed=1, sigma=sig)
cfg = G.SketchConfig(strategy=G.Strategy.Gaussian, size=l, seed=o.derive(1, 0x5E7C))
f, _, _ = G._factor(_abi.RLU, a, cfg, _abi.options(diagnostics=True))
out = {"m": m, "n": n, "l": l, "gpu": {"orth": G.orthogonality_error_dev(f.q), "res": G.residual_error_dev(a, f.q, f.r),
                                       "cond_x": f.report.stages[1].cond_x}}
ah = np.ascontiguousarray(a.cpu().numpy())
qg = f.q.cpu().numpy()
del a, f
torch.cuda.empty_cache()
o.set_test_threads(os.cpu_count())
t0 = time.time()
ref = o.factor(_abi.RLU, ah, cfg._c(), _abi.options(), workers=os.cpu_count())
out["oracle_s"] = time.time() - t0
out["oracle"] = {"orth": o.orthogonality_error(ref.q), "res": o.residual_error(ah, ref.q, ref.r)}
out["gpu_orth_by_oracle_diag"] = o.orthogonality_error(qg)
out["dQ"] = float(np.linalg.norm(qg - ref.q) / np.sqrt(n))
print(json.dumps(out))
