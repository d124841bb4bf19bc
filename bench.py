"""bench.py — rQR/rLU-CholeskyQR fp64 on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[1], "c1"): rLU-CholeskyQR, m = 1,000,000 rows
per GPU, n = 128, Gaussian sketch s = 2n = 256, A = U diag(sigma) V^T with
sigma log-spaced 1 .. 1e-14 (cond 1e14). Synthetic, seeded; U from a QR of a
torch Gaussian on the device, V from a numpy QR (input generation is outside
the timed region). N > 1: weak scaling, one 1e6-row block per rank
(parexec.cpp:9-18), partials summed with NCCL.

One step = one full factorization (sketch, LU, two trisolves, Gram, Cholesky,
recover) through the C-ABI on the HBM-resident A. value = algorithmic TFLOP/s
of the whole job; ms_per_step = ms per factorization.

--impl reference: the CPU oracle port of the reference (oracle/, the
reference itself cannot be built here: no Eigen) on the host cores, rank 0
only, on a bounded row sample of the same workload.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

M_PER_GPU = 1_000_000
N = 128
RATE = 2.0
KAPPA = 1e14
SEED = 1
CPU_SAMPLE_ROWS = 100_000
WORKLOAD = "c1: rLU-CholeskyQR fp64, m=1e6 rows/GPU, n=128, Gaussian sketch s=256, cond 1e14"
# BASELINE.json configs (per-GPU shapes; c1 is the benchmark line, the others via --workload):
# name -> (method name, m per GPU, n, sketch rows l, kappa or "two-segment", description)
WORKLOADS = {
    "c1": ("rlu", M_PER_GPU, N, 256, KAPPA, WORKLOAD),
    "c2": ("rqr-gaussian", 4_000_000, 256, 512, 1e12,
           "c2: rQR-CholeskyQR (Gaussian) fp64, m=4e6 rows/GPU, n=256, s=512, cond 1e12"),
    "c3": ("rqr-gaussian", 4_194_304, 64, 128, 1e15,
           "c3: rQR-CholeskyQR (Gaussian) fp64, m=4194304 rows/GPU, n=64, s=128, cond 1e15"),
    "c4": ("rlu", 1_000_000, 512, 768, "two-segment",
           "c4: rLU-CholeskyQR (Gaussian) fp64, m=1e6 rows/GPU, n=512, s=768, sigma 10^(-8i/255) then 1e-8"),
}


def workload_sigma(n, kappa):
    import numpy as np

    if kappa == "two-segment":  # BASELINE.json c4
        s = np.full(n, 1e-8)
        s[:256] = 10.0 ** (-8.0 * np.arange(256) / 255.0)
        return s
    from paper_2111_11148_b200 import cholqr as cq

    return cq.geometric_sigma(n, kappa)


def flops_rlu(m, n, l):
    """Algorithmic flops of one rLU-CholeskyQR factorization."""
    tall = 2.0 * l * m * n + 2.0 * m * n * n + m * n * (n + 1)
    small = (l * n * n - n ** 3 / 3.0) + n ** 3 / 3.0 + n ** 3 / 3.0  # LU, Cholesky, recover
    return tall + small


def peaks():
    p = {"hbm_gbs": None, "fp64_tflops": 37.1, "fp64_src": "measured DMMA m8n8k4 peak, tools/probe/fp64_probe.cu "
         "(profiles/r01_fp64_probe.txt); MEASURED_PEAKS.json has no FP64 entry"}
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        p["hbm_gbs"] = mp.get("hbm_gbs")
    except Exception:
        p["hbm_gbs"] = 6650.0
    return p


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def make_input(m_local, n, rank, world, device, kappa=None, ctx=None, sigma=None):
    """Rows [rank*m_local, (rank+1)*m_local) of A = U diag(sigma) V^T, generated on
    the device by the library (matgen.cpp:21-46 restated: counter-RNG Gaussians,
    seeds derive(SEED, 0/1), orthonormalised across all ranks)."""
    from paper_2111_11148_b200 import cholqr as cq

    if ctx is None:
        from paper_2111_11148_b200 import dist

        ctx = dist.make_context(device.index if hasattr(device, "index") else int(device), rank, world)
    k = KAPPA if kappa is None else kappa
    return cq.synthesize_dev(m_local, n, k, SEED, sigma=sigma, device=ctx.device, m_global=m_local * world,
                             row0=rank * m_local, ctx=ctx)


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as td

    from paper_2111_11148_b200 import _abi
    from paper_2111_11148_b200 import cholqr as cq
    from paper_2111_11148_b200 import dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        td.init_process_group("nccl", device_id=dev)
    ctx = dist.make_context(local, rank, world)
    mname, m_local, n, l_req, kap, wdesc = WORKLOADS[args.workload]
    method = {v: k for k, v in _abi.METHOD_NAMES.items()}[mname]
    m_global = m_local * world
    row0 = rank * m_local
    a = make_input(m_local, n, rank, world, dev, ctx=ctx, sigma=workload_sigma(n, kap))
    q = torch.empty_like(a)
    cfg = cq.SketchConfig(strategy=cq.Strategy.Gaussian, size=l_req, rate=RATE, seed=_seed_value())
    l = cfg.resolved_size(m_global, n)
    opts = _abi.options()

    def step():
        return dist.factor_sharded(ctx, method, a, m_global, row0, cfg, opts, q_out=q)

    for _ in range(args.warmup):
        step()
    # correctness of the benchmarked factorization (outside the timed region)
    _, r, rep = step()
    orth = cq.orthogonality_error_dev(q, ctx)  # sharded: Gram of Q summed over the ranks
    res = cq.residual_error_dev(a, q, r, ctx)

    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sketch_ms, stage_tot = [], np.zeros(_abi.STAGE_COUNT)
    if world > 1:
        td.barrier()
    torch.cuda.synchronize(dev)
    l0 = ctx.launches
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            _, _, rep = step()
            sketch_ms.append(rep.stage_ms[0])
            stage_tot += np.array(rep.stage_ms[:])
        e1.record(stream)
        torch.cuda.synchronize(dev)
    launches = ctx.launches - l0
    if world > 1:
        td.barrier()
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], device=dev, dtype=torch.float64)
    if world > 1:
        td.all_reduce(t, op=td.ReduceOp.MAX)
    ms = float(t.item())
    ms_step = ms / args.steps
    total_flops = flops_rlu(m_global, n, l)
    value = total_flops / (ms_step * 1e-3) / 1e12

    # e2e through the public host-buffer API (H2D of A, factorization, D2H of Q and R):
    # cqr_factor on one GPU, cqr_factor_sharded (this rank's rows) on several
    ah = a.cpu().pin_memory()
    qh = torch.empty_like(ah).pin_memory()
    rh = np.zeros((n, n))
    an, qn = ah.numpy(), qh.numpy()
    rep2 = _abi.Report()
    cfg_c = cfg._c()

    def e2e_step():
        import ctypes as C
        if world == 1:
            st = cq._lib().cqr_factor(ctx.h, method, C.c_void_p(an.ctypes.data), m_local, n, n, C.byref(cfg_c),
                                      C.byref(opts), C.c_void_p(qn.ctypes.data), n, cq._ptr(rh), n, C.byref(rep2))
        else:
            st = cq._lib().cqr_factor_sharded(ctx.h, method, C.c_void_p(an.ctypes.data), m_local, m_global, row0,
                                              n, n, C.byref(cfg_c), C.byref(opts), C.c_void_p(qn.ctypes.data), n,
                                              cq._ptr(rh), n, C.byref(rep2))
        ctx._check(st, rep2.index)

    e2e_step()
    ke = max(3, min(args.steps, 10))
    if world > 1:
        td.barrier()
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for _ in range(ke):
        e2e_step()
    torch.cuda.synchronize(dev)
    te = torch.tensor([(time.perf_counter() - t0) / ke], device=dev, dtype=torch.float64)
    if world > 1:
        td.all_reduce(te, op=td.ReduceOp.MAX)
    te = float(te.item())
    e2e = {"value": total_flops / te / 1e12, "unit": "TFLOP/s", "ms_per_step": te * 1e3,
           "h2d_bytes_per_step": int(8 * m_global * n), "d2h_bytes_per_step": int(8 * m_global * n + 8 * n * n * world),
           "api": "cqr_factor (host pinned buffers)" if world == 1 else
                  "cqr_factor_sharded per rank (host pinned buffers), max over ranks"}

    pk = peaks()
    sk_ms = statistics.mean(sketch_ms)
    sk_flops = 2.0 * l * m_local * n
    achieved = sk_flops / (sk_ms * 1e-3) / 1e12
    roof = {"kernel": "sketch_ws_kernel (8 Box-Muller warps + 8 DMMA warps) + sketch_reduce (Sketch stage)",
            "bound": "tensor",
            "achieved": achieved, "peak": pk["fp64_tflops"], "unit": "TFLOP/s", "frac": achieved / pk["fp64_tflops"],
            "peak_src": pk["fp64_src"], "algorithmic": f"2*l*m*n flops per launch (l={l}, m={m_local}, n={n}); "
            "Omega generation (l*m Gaussian draws) is extra work not counted",
            "traffic": _traffic() if args.workload == "c1" else None}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline_sample(a, l, CPU_SAMPLE_ROWS, method, mname)
    stage_avg = {cq_name: float(v / args.steps) for cq_name, v in zip(_abi.STAGE_NAMES, stage_tot)}
    # per stage: algorithmic flops of this rank's part / CUDA-event stage time, vs the DMMA peak
    qr = mname.startswith("rqr")
    st_flops = {"sketch": 2.0 * l * m_local * n, "precondition": (2.0 if qr else 1.0) * (l * n * n - n ** 3 / 3.0),
                "gram": float(m_local) * n * (n + 1), "cholesky": n ** 3 / 3.0, "trisolve": 2.0 * m_local * n * n,
                "recover": n ** 3 / 3.0}
    stage_roof = {k: {"tflops": f / (stage_avg[k] * 1e-3) / 1e12, "frac": f / (stage_avg[k] * 1e-3) / 1e12 /
                      pk["fp64_tflops"]} for k, f in st_flops.items() if stage_avg.get(k, 0.0) > 0.0}
    line = {"metric": "rQR/rLU-CholeskyQR fp64 TFLOP/s (ms/factorization in ms_per_step)", "value": value,
            "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: A = U diag(sigma) V^T generated on the device (matgen.cpp restated), "
                    + ("sigma log-spaced 1..1/kappa" if kap != "two-segment" else "c4 two-segment spectrum"),
            "config": {"workload": wdesc, "method": mname, "sketch": "gaussian", "m_per_gpu": m_local,
                       "m_global": m_global, "n": n, "l": l, "kappa": kap,
                       "l2": f"inputs larger than L2 ({8 * m_local * n / 1e9:.2f} GB per GPU vs 126 MB L2), no flush",
                       "parallelism": f"row-block dp{world}"},
            "stage_ms": stage_avg, "clocks": clk.summary(), "gpu_launches": launches,
            "roofline": roof, "stage_roofline": stage_roof, "cpu_baseline": cpu, "e2e": e2e,
            "check": {"orth": orth, "res": res, "sketch_rows": rep.sketch_rows}}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        td.destroy_process_group()


def _traffic():
    p = os.path.join(ROOT, "profiles", "sketch_traffic.json")
    try:
        return json.load(open(p))["bytes_per_launch"]
    except Exception:
        return None


def cpu_baseline_sample(a_dev, l, rows, method=None, mname="rlu"):
    """Oracle (CPU port of the reference) on the first `rows` rows of the same A."""
    import numpy as np

    from oracle import oracle as o
    from paper_2111_11148_b200 import _abi

    a = np.ascontiguousarray(a_dev[:rows].cpu().numpy())
    cores = os.cpu_count() or 1
    cfg = _abi.sketch_cfg(strategy=_abi.GAUSSIAN, size=l, rate=RATE, seed=_seed_value())
    t0 = time.perf_counter()
    o.factor(_abi.RLU if method is None else method, a, cfg, _abi.options(), workers=cores)
    dt = time.perf_counter() - t0
    fl = flops_rlu(rows, a.shape[1], l)
    return {"value": fl / dt / 1e12, "unit": "TFLOP/s", "cores": cores, "kind": "port",
            "sample": f"one {mname} factorization of the first {rows} rows (n={a.shape[1]}, l={l}); "
                      f"{dt:.2f} s; sketch serial as in sketch.cpp:94-116, Gram/trisolve on {cores} workers"}


def _seed_value():
    # derive(SEED, 0x5E7C) (experiments.cpp:94), computed with the product's own host RNG
    m64 = (1 << 64) - 1

    def mix(z):
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m64
        return z ^ (z >> 31)

    return mix(SEED ^ mix((0x5E7C + 0x51ED270B8A5EC473) & m64))


def run_reference(args):
    """--impl reference: the oracle port on all host cores, rank 0 only."""
    import numpy as np

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import oracle as o
    from paper_2111_11148_b200 import _abi

    mname, _, n, l, kap, wdesc = WORKLOADS[args.workload]
    method = {v: k for k, v in _abi.METHOD_NAMES.items()}[mname]
    rows = CPU_SAMPLE_ROWS
    rs = np.random.default_rng(SEED)
    u, _ = np.linalg.qr(rs.standard_normal((rows, n)))
    v, _ = np.linalg.qr(rs.standard_normal((n, n)))
    sigma = workload_sigma(n, kap)
    a = np.ascontiguousarray(u @ (sigma[:, None] * v.T))
    cores = os.cpu_count() or 1
    cfg = _abi.sketch_cfg(strategy=_abi.GAUSSIAN, size=l, rate=RATE, seed=_seed_value())
    for _ in range(args.warmup):
        o.factor(method, a, cfg, _abi.options(), workers=cores)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        o.factor(method, a, cfg, _abi.options(), workers=cores)
    dt = (time.perf_counter() - t0) / args.steps
    value = flops_rlu(rows, n, l) / dt / 1e12
    line = {"impl": "reference", "metric": "rQR/rLU-CholeskyQR fp64 TFLOP/s (ms/factorization in ms_per_step)",
            "value": value, "unit": "TFLOP/s", "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": wdesc, "method": mname, "sketch": "gaussian", "n": n, "l": l,
                       "kappa": kap, "sample_rows": rows},
            "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": cores, "kind": "port",
                             "sample": f"{mname} of a {rows} x {n} sample per step (the reference is "
                                       "not buildable here: no Eigen); serial Gaussian sketch as the reference"},
            "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    ap.add_argument("--workload", default="c1", choices=sorted(WORKLOADS),
                    help="BASELINE.json config (c1, the benchmark line, by default)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
