import sys, numpy as np
sys.path.insert(0, '/root/repo')
from oracle import oracle as o
from paper_2111_11148_b200 import cholqr as G
U = 2.0 ** -52
worst, same, tot = 0.0, 0, 0
for seed in (0, 1, 42, 7, 99):
    n = 2_000_000
    gd = G.rng_gaussian(seed, 1000, n)
    go = o.gaussian_fill(seed, 1000, n)
    err = np.abs(gd - go) / (U * np.maximum(np.abs(go), 1.0))
    worst = max(worst, err.max()); same += int((gd == go).sum()); tot += n
print(f"max err {worst:.2f} ulp(max(|g|,1)), bit-identical {same / tot:.4f}")
