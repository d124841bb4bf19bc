"""Trisolve A/B: time X R = A at (m, n) for the kernel variant selected by CQR_TRISOLVE_VARIANT
(0: default dispatch, 2: left-looking TMA kernel) and save X for a bitwise comparison across runs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as o  # noqa: E402
from paper_2111_11148_b200 import cholqr as cq  # noqa: E402

m, n = int(sys.argv[1]), int(sys.argv[2])
tag = os.environ.get("CQR_TRISOLVE_VARIANT", "0")
g = torch.Generator(device="cuda").manual_seed(5)
a = torch.randn(m, n, dtype=torch.float64, device="cuda", generator=g)
r = torch.as_tensor(o.qr_r_factor(o.gaussian_matrix(2 * n, n, 3)), device="cuda")
x = a.clone()
cq.right_trisolve_in_place(x, r)
out = f"/tmp/tri_{m}_{n}_{tag}.npy"
np.save(out, x.cpu().numpy())
for _ in range(3):
    x.copy_(a)
    cq.right_trisolve_in_place(x, r)
ts = []
for _ in range(7):
    x.copy_(a)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    cq.right_trisolve_in_place(x, r)
    e.record()
    torch.cuda.synchronize()
    ts.append(s.elapsed_time(e))
ms = sorted(ts)[len(ts) // 2]
print(f"variant {tag} m={m} n={n}: {ms:.3f} ms/call ({m * n * n / ms / 1e9:.1f} TFLOP/s incl. pack+sync)", flush=True)
if tag != "2" and os.path.exists(f"/tmp/tri_{m}_{n}_2.npy"):
    ref = np.load(f"/tmp/tri_{m}_{n}_2.npy")
    print("  bitwise equal to the left-looking kernel:", np.array_equal(ref, np.load(out)), flush=True)
