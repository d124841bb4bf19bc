import sys, statistics
sys.path.insert(0, "/root/repo")
from paper_2111_11148_b200 import _abi
from paper_2111_11148_b200 import cholqr as G
m, n = 1_000_000, 100
a = G.synthesize_dev(m, n, 1e5, 1)
FIXED = G.ShiftMode.fixed(1e-15) if hasattr(G.ShiftMode, "fixed") else None
for method in (_abi.RQR, _abi.CHOLQR2):
    for rnd in range(4):
        cfg = G.SketchConfig(seed=10 + rnd)
        _, timing, _ = G._factor(method, a, cfg, G._opts(G.Options()))
    print(_abi.METHOD_NAMES[method], round(timing.total_ms, 3), [round(x, 3) for x in timing.stage_ms])
