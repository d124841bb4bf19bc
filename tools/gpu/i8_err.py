import os, sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_2111_11148_b200 import cholqr as G, _abi
from oracle import oracle as o
m, n, l = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
a = G.synthesize_dev(m, n, 1e10, 1).cpu().numpy()
sk = G.sketch_gaussian(a, G.SketchConfig(strategy=G.Strategy.Gaussian, size=l, seed=5)).a1
o.set_test_threads(16)
ref = o.sketch_gaussian(a, l, 5)
err = np.abs(sk - ref)
print("rel fro", np.linalg.norm(sk - ref) / np.linalg.norm(ref))
print("max err per column (first 8, last 8):", err.max(0)[:8], err.max(0)[-8:])
print("max err per row (first 8):", err.max(1)[:8])
print("scale", np.abs(ref).max(), "worst col", err.max(0).argmax(), "worst row", err.max(1).argmax())
# relative to sum |w||a|
