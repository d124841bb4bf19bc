"""bench.py — rQR/rLU-CholeskyQR fp64 on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[1], "c1", the default): rLU-CholeskyQR with a
Gaussian sketch, m = 1,000,000 rows per GPU, n = 128, s = 2n = 256,
A = U diag(sigma) V^T with sigma log-spaced 1 .. 1e-14 (cond 1e14). Synthetic
and seeded: A is generated on the device by the library's matgen
(cqr_synthesize_dev, matgen.cpp:21-46 restated: counter-RNG Gaussians from
derive(1, 0/1), orthonormalised); the sketch seed is derive(1, 0x5E7C)
(experiments.cpp:94). Input generation is outside the timed region.

  --workload c2   rQR-Gaussian, m = 4e6 FIXED, n = 256, s = 512, cond 1e12: strong
                  scaling, rank b owns rows [ceil(b m/p), ceil((b+1) m/p)) (parexec.cpp:13-15)
  --workload c3   rQR-Gaussian, 4,194,304 rows PER GPU, n = 64, s = 128, cond 1e15: weak scaling
  --workload c4   rLU-Gaussian, m = 1e6, n = 512, s = 768, two-segment sigma (strong)
  c1              1e6 rows per GPU (weak) -- BASELINE.json runs it on 1 B200

One step = one full factorization (sketch, LU/QR, two trisolves, Gram,
Cholesky, recover) through the C-ABI on the HBM-resident A. value = algorithmic
TFLOP/s of the whole job (all ranks); ms_per_step = ms per factorization (max
over ranks, CUDA events on the library's stream). e2e = the same factorization
through the host-buffer C-ABI (cqr_factor / cqr_factor_sharded): H2D of A and
D2H of Q and R inside the timed region.

--gpus N without WORLD_SIZE in the environment re-launches this script under
torch.distributed.run (one process per GPU, 127.0.0.1, NCCL_DEBUG=INFO so the
log shows the ranks); with WORLD_SIZE set it must equal N.

--impl reference: the CPU oracle port of the reference (oracle/; the reference
itself cannot be built here or on the GPU box: no Eigen) on the host cores,
rank 0 only, on a bounded row sample of the same workload per step.
"""
import argparse
import json
import os
import platform
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N = 128
RATE = 2.0
KAPPA = 1e14
SEED = 1
REF_SAMPLE_ROWS = 100_000  # --impl reference: rows of the per-step CPU sample
METRIC = "rQR/rLU-CholeskyQR fp64 TFLOP/s (ms/factorization in ms_per_step)"
# BASELINE.json configs: name -> (method, rows, per_gpu (weak) or fixed global (strong), n, l, kappa, description)
WORKLOADS = {
    "c1": ("rlu", 1_000_000, True, N, 256, KAPPA,
           "c1: rLU-CholeskyQR (Gaussian) fp64, m=1e6 rows/GPU, n=128, s=256, cond 1e14"),
    "c2": ("rqr-gaussian", 4_000_000, False, 256, 512, 1e12,
           "c2: rQR-CholeskyQR (Gaussian) fp64, m=4e6 (fixed, row blocks ceil(b*m/p)), n=256, s=512, cond 1e12"),
    "c3": ("rqr-gaussian", 4_194_304, True, 64, 128, 1e15,
           "c3: rQR-CholeskyQR (Gaussian) fp64, m=4194304 rows/GPU, n=64, s=128, cond 1e15"),
    "c4": ("rlu", 1_000_000, False, 512, 768, "two-segment",
           "c4: rLU-CholeskyQR (Gaussian) fp64, m=1e6, n=512, s=768, sigma 10^(-8i/255) then 1e-8"),
}
FP64_PEAK = {"value": 37.1, "src": "builder-measured: DMMA m8n8k4 FP64 peak of this B200 pool "
             "(tools/probe/fp64_probe.cu, profiles/r01_fp64_probe.txt); MEASURED_PEAKS.json has no FP64 entry"}
# The sketch runs as an exact integer product on the int8 tensor cores (csrc/sketch_i8.cu): 28 int8 MACs per
# FP64 MAC (7 balanced byte digits per operand, levels s + t <= 6). Its roof in FP64-equivalent terms is the
# measured int8 tcgen05 rate / 28: 8181 MAC/clk/SM (tools/probe/umma_i8.cu, M=128 N=256 K=32, profiles/
# r02_umma_i8_probe.txt) x 148 SMs x 1.965 GHz = 2.38e15 MAC/s -> 8.50e13 FP64-equivalent MAC/s = 170 TFLOP/s.
I8_EMU_PEAK = {"value": 2.0 * 8181 * 148 * 1.965e9 / 28 / 1e12,
               "src": "builder-measured int8 tcgen05 MMA rate (tools/probe/umma_i8.cu: 8181 MAC/clk/SM at N=256) "
                      "x 148 SMs x 1.965 GHz / 28 int8 MACs per FP64-equivalent MAC; MEASURED_PEAKS.json has "
                      "no int8 entry"}


def workload_sigma(n, kappa):
    import numpy as np

    if kappa == "two-segment":  # BASELINE.json configs[4]
        s = np.full(n, 1e-8)
        s[:256] = 10.0 ** (-8.0 * np.arange(256) / 255.0)
        return s
    sig = np.ones(n)
    if n > 1:  # matgen.cpp:27-31
        sig[1:] = np.exp(-np.log(kappa) * np.arange(1, n) / (n - 1))
    return sig


def flops_factorization(method, m, n, l):
    """Algorithmic flops of one rQR/rLU-CholeskyQR factorization: sketch
    2lmn, two tall solves 2mn^2, Gram mn(n+1), plus the small factorizations."""
    tall = 2.0 * l * m * n + 2.0 * m * n * n + m * n * (n + 1)
    pre = (2.0 if method.startswith("rqr") else 1.0) * (l * n * n - n ** 3 / 3.0)  # QR 2n^2(l-n/3), LU n^2(l-n/3)
    return tall + pre + n ** 3 / 3.0 + n ** 3 / 3.0  # + Cholesky + recover


def flops_cholqr_family(method, m, n):
    passes = {"cholqr": 1, "cholqr2": 2, "scholqr3": 3}[method]
    return passes * (m * n * (n + 1) + m * n * n + n ** 3 / 3.0) + (passes - 1) * n ** 3 / 3.0


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region: NVML in a thread of this
    process every 5 ms (a factorization is a few ms, the timed region ~0.1 s; an nvidia-smi child
    every 100 ms caught a single sample), nvidia-smi as the fallback."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device):
        self.device = device
        self.rows = []  # (sm_mhz, sm_max_mhz, [active reason names])
        self.proc = None
        self.stop = threading.Event()
        self.src = None

    def _nvml_handle(self):
        import pynvml as nv

        nv.nvmlInit()
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        idx = self.device
        if vis:
            ent = vis.split(",")[self.device].strip()
            if not ent.isdigit():
                return nv, nv.nvmlDeviceGetHandleByUUID(ent)
            idx = int(ent)
        return nv, nv.nvmlDeviceGetHandleByIndex(idx)

    def _sample_nvml(self):
        nv, h = self.nv, self.h
        bits = [(nv.nvmlClocksEventReasonHwSlowdown, 0), (nv.nvmlClocksEventReasonHwThermalSlowdown, 1),
                (nv.nvmlClocksEventReasonSwThermalSlowdown, 2), (nv.nvmlClocksEventReasonSwPowerCap, 3)]
        try:
            sm = float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
            mask = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            self.rows.append((sm, self.mx, [self.NAMES[i] for b, i in bits if mask & b]))
        except Exception:
            pass

    def _poll_nvml(self):
        while not self.stop.is_set():
            self._sample_nvml()
            self.stop.wait(0.005)

    def _read_smi(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6 and parts[0].replace(".", "").isdigit() and parts[1].replace(".", "").isdigit():
                self.rows.append((float(parts[0]), float(parts[1]),
                                  [self.NAMES[i] for i in range(4) if parts[2 + i].lower().startswith("active")]))

    def __enter__(self):
        try:
            # the slow first NVML calls happen here, not in the sampling thread (a 50 ms region once ended before
            # the thread's first sample); the first sample is taken right after the warm-up steps, the last one
            # right after the region's last step, so there are always at least two
            self.nv, self.h = self._nvml_handle()
            self.mx = float(self.nv.nvmlDeviceGetMaxClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            self._sample_nvml()
            if not self.rows:
                raise RuntimeError("nvml sample failed")
            self.src = "nvml"
            self.t = threading.Thread(target=self._poll_nvml, daemon=True)
            self.t.start()
            return self
        except Exception:
            pass
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.src = "nvidia-smi"
            self.t = threading.Thread(target=self._read_smi, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.stop.set()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        elif self.src == "nvml":
            self.t.join(timeout=1)
            self._sample_nvml()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(r[0] for r in self.rows), "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": sorted({x for r in self.rows for x in r[2]}), "samples": len(self.rows),
                "source": self.src}


def shard(m_global, world, rank):
    """(row0, rows) of rank's block, ceil(b*m/p) offsets (parexec.cpp:13-15)."""
    lo = -(-rank * m_global // world)
    hi = -(-(rank + 1) * m_global // world)
    return lo, hi - lo


def workload_shape(name, world, rank, rows_override=None):
    mname, rows, weak, n, l, kap, desc = WORKLOADS[name]
    if rows_override:
        rows, desc = rows_override, desc + f" [--rows {rows_override}: a flow check, not the workload]"
    m_global = rows * world if weak else rows
    row0, m_local = shard(m_global, world, rank)
    return mname, m_global, row0, m_local, n, l, kap, desc, weak


def traffic_for(workload):
    """dram read+write bytes per launch of the workload's dominant kernel, from the
    committed ncu capture (profiles/traffic.json, written by tools/traffic_summary.py)."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        return d[workload]
    except Exception:
        return None


def run_ours(args):
    import ctypes as C

    import numpy as np
    import torch
    import torch.distributed as td

    from paper_2111_11148_b200 import _abi
    from paper_2111_11148_b200 import cholqr as cq
    from paper_2111_11148_b200 import dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    host_tr = args.transport == "host" and world > 1
    if host_tr:
        # ranks share the visible GPUs round-robin; the exchange steps go through pinned host buffers
        # and gloo (dist.HostTransport). No kernel waits on another rank, so this is safe on one GPU;
        # it validates the N-rank flow, its timings are not scaling numbers.
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    rdev = torch.device("cpu") if host_tr else dev  # where the max-over-ranks scalars live
    if host_tr:
        td.init_process_group("gloo")
        ctx = cq.Context(local)
        dist.attach_host_transport(ctx)
    else:
        if world > 1:
            td.init_process_group("nccl", device_id=dev)
        ctx = dist.make_context(local, rank, world)
    mname, m_global, row0, m_local, n, l_req, kap, wdesc, weak = workload_shape(args.workload, world, rank, args.rows)
    method = {v: k for k, v in _abi.METHOD_NAMES.items()}[mname]
    a = cq.synthesize_dev(m_local, n, seed=SEED, sigma=workload_sigma(n, kap), m_global=m_global, row0=row0,
                          ctx=ctx)
    q = torch.empty_like(a)
    cfg = cq.SketchConfig(strategy=cq.Strategy.Gaussian, size=l_req, rate=RATE, seed=cq.derive(SEED, 0x5E7C))
    l = cfg.resolved_size(m_global, n)
    opts = _abi.options()
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)

    def step():
        return dist.factor_sharded(ctx, method, a, m_global, row0, cfg, opts, q_out=q)

    for _ in range(args.warmup):
        step()
    # correctness of the benchmarked factorization (outside the timed region)
    _, r, rep = step()
    orth = cq.orthogonality_error_dev(q, ctx)  # sharded: Gram of Q summed over the ranks
    res = cq.residual_error_dev(a, q, r, ctx)

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
    t = torch.tensor([ms], device=rdev, dtype=torch.float64)
    if world > 1:
        td.all_reduce(t, op=td.ReduceOp.MAX)
    ms_step = float(t.item()) / args.steps
    total_flops = flops_factorization(mname, m_global, n, l)
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
    te = torch.tensor([(time.perf_counter() - t0) / ke], device=rdev, dtype=torch.float64)
    if world > 1:
        td.all_reduce(te, op=td.ReduceOp.MAX)
    te = float(te.item())
    e2e = {"value": total_flops / te / 1e12, "unit": "TFLOP/s", "ms_per_step": te * 1e3,
           "h2d_bytes_per_step": int(8 * m_global * n), "d2h_bytes_per_step": int(8 * m_global * n + 8 * n * n * world),
           "api": "cqr_factor (host pinned buffers)" if world == 1 else
                  "cqr_factor_sharded per rank (host pinned buffers), max over ranks",
           "timer": "host wall clock around blocking calls, max over ranks"}

    if world == 1 and args.workload == "c1" and not args.no_overlap:
        e2e["two_in_flight"] = e2e_two_in_flight(local, method, an, qn, m_local, n, cfg, ke, total_flops)

    sk_ms = statistics.mean(sketch_ms)
    sk_flops = 2.0 * l * m_local * n
    achieved = sk_flops / (sk_ms * 1e-3) / 1e12
    traffic = traffic_for(args.workload)
    roof = {"kernel": "sketch_i8_kernel (Omega drawn in-kernel, A1 = Omega A as an exact int8 tcgen05 product, "
                      "the column exponent scan in-kernel) + the fixed-order reduce (Sketch stage events)",
            "bound": "tensor", "achieved": achieved, "peak": FP64_PEAK["value"], "unit": "TFLOP/s",
            "frac": achieved / FP64_PEAK["value"],
            "peak_src": FP64_PEAK["src"] + " (north_star: the binding roofline is FP64 compute or HBM; the sketch "
                        "delivers FP64-accurate Omega A, so its flops are counted against the chip's FP64 roof)",
            "frac_note": "the FP64-equivalent rate can reach or pass the DMMA peak: the exact product runs on the "
                         "int8 tensor cores, whose own roof (int8_emulation) is ~4.6x higher; the kernel is bound by "
                         "the in-kernel Box-Muller draws of Omega",
            "int8_emulation": {"peak": I8_EMU_PEAK["value"], "frac": achieved / I8_EMU_PEAK["value"],
                               "peak_src": I8_EMU_PEAK["src"],
                               "note": "the same flops against the roof of the int8 tensor-core emulation the "
                                       "kernel runs (28 int8 MACs per FP64 MAC); the kernel is bound below it by "
                                       "the in-kernel Box-Muller draws of Omega"},
            "algorithmic": f"2*l*m*n FP64-equivalent flops per launch (l={l}, m={m_local}, n={n}); the l*m "
                           "Box-Muller draws of Omega (the kernel's actual bound: issue-limited generator warps, "
                           "DESIGN.md 4) are extra work, not counted",
            "traffic": traffic["bytes_per_launch"] if traffic and "sketch" in traffic["kernel"] else None,
            "traffic_vs_algorithmic": (traffic["bytes_per_launch"] / (8.0 * m_local * n)
                                       if traffic and "sketch" in traffic["kernel"] else None),
            "traffic_note": "A is read twice by design: the scanner warps find each sub-chunk's exponent bounds one "
                            "sub-chunk ahead of the TMA stream that feeds the slicers (the kernel is bound by the "
                            "Box-Muller draws, not HBM: 2 x 8mn bytes in the kernel's time is ~1.2 TB/s)"}
    tri_ms = float(stage_tot[_abi.STAGE_NAMES.index("trisolve")] / args.steps / 2.0)  # two solves per factorization
    if traffic and "trisolve" in traffic["kernel"]:
        # the dominant kernel of this workload (profiles/traffic.json, from the committed launch list) is the solve
        tflops = float(m_local) * n * n / (tri_ms * 1e-3) / 1e12
        roof = {"kernel": f"{traffic['kernel']} (per call: Trisolve stage / 2, CUDA events)", "bound": "tensor",
                "achieved": tflops, "peak": FP64_PEAK["value"], "unit": "TFLOP/s", "frac": tflops / FP64_PEAK["value"],
                "peak_src": FP64_PEAK["src"],
                "algorithmic": f"m*n^2 flops per launch (m={m_local}, n={n}): the off-block terms on DMMA, the "
                               "diagonal recurrence on the FP64 pipe; 16 m n bytes algorithmic",
                "traffic": traffic["bytes_per_launch"], "traffic_vs_algorithmic": traffic["bytes_per_launch"] /
                (16.0 * m_local * n), "sketch": {k: v for k, v in roof.items() if k != "traffic"}}
    stage_avg = {nm: float(v / args.steps) for nm, v in zip(_abi.STAGE_NAMES, stage_tot)}
    # per stage: algorithmic flops of this rank's part / CUDA-event stage time, vs the DMMA peak
    qr = mname.startswith("rqr")
    st_flops = {"sketch": 2.0 * l * m_local * n, "precondition": (2.0 if qr else 1.0) * (l * n * n - n ** 3 / 3.0),
                "gram": float(m_local) * n * (n + 1), "cholesky": n ** 3 / 3.0, "trisolve": 2.0 * m_local * n * n,
                "recover": n ** 3 / 3.0}
    stage_roof = {k: {"tflops": f / (stage_avg[k] * 1e-3) / 1e12, "frac": f / (stage_avg[k] * 1e-3) / 1e12 /
                      FP64_PEAK["value"]} for k, f in st_flops.items() if stage_avg.get(k, 0.0) > 0.0}

    comparison = None
    if args.workload == "c1" and not args.no_compare:
        comparison = compare_methods(ctx, a, m_global, row0, n, args, stream, dev, world, rdev)

    cpu = None
    if not args.no_cpu:
        # the oracle on the whole c1 A of rank 0 (the same bytes), after the timed regions
        cpu = cpu_baseline(a, m_local, n, l, method, mname) if (rank == 0 and args.workload == "c1") else None
    if world > 1:
        td.barrier()
    line = {"metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak" if weak else "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: A = U diag(sigma) V^T generated on the device (matgen.cpp restated), "
                    + ("sigma log-spaced 1..1/kappa" if kap != "two-segment" else "c4 two-segment spectrum"),
            "config": {"workload": wdesc, "method": mname, "sketch": "gaussian", "m_global": m_global,
                       "m_per_gpu": m_local if weak else None, "n": n, "l": l, "kappa": kap,
                       "l2": f"inputs larger than L2 ({8 * m_local * n / 1e9:.2f} GB per GPU vs 126 MB L2), no flush",
                       "parallelism": f"row-block dp{world}" + ("" if weak else " (strong: fixed m, ceil(b*m/p) blocks)"),
                       "transport": ("host (gloo + pinned staging; ranks may share a GPU: a flow check, not a "
                                     "scaling number)" if host_tr else "nccl" if world > 1 else None)},
            "stage_ms": stage_avg, "clocks": clk.summary(), "gpu_launches": launches,
            "roofline": roof, "stage_roofline": stage_roof, "cpu_baseline": cpu, "e2e": e2e,
            "comparison": comparison,
            "check": {"orth": orth, "res": res, "sketch_rows": rep.sketch_rows}}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        td.destroy_process_group()


def e2e_two_in_flight(device, method, an, qn, m, n, cfg, ke, flops):
    """Extra to e2e (not the headline): the same blocking cqr_factor calls issued from TWO host threads, each
    on its own context (cqr.h: one context per thread) and its own pinned buffers, so one call's D2H of Q
    overlaps the other's H2D of A on the full-duplex link. Every step still moves its A in and its Q, R out
    inside the timed region; the number is factorizations completed per wall-clock second."""
    import ctypes as C
    import threading

    import numpy as np
    import torch

    from paper_2111_11148_b200 import _abi
    from paper_2111_11148_b200 import cholqr as cq

    errs, start = [], threading.Barrier(3)
    bufs = [(an, qn)]
    a2 = torch.from_numpy(an).clone().pin_memory()
    q2 = torch.empty_like(a2).pin_memory()
    bufs.append((a2.numpy(), q2.numpy()))

    def worker(i):
        try:
            ctx = cq.Context(device)
            a_h, q_h = bufs[i]
            r_h, rep, cfg_c, opts = np.zeros((n, n)), _abi.Report(), cfg._c(), _abi.options()

            def one():
                st = cq._lib().cqr_factor(ctx.h, method, C.c_void_p(a_h.ctypes.data), m, n, n, C.byref(cfg_c),
                                          C.byref(opts), C.c_void_p(q_h.ctypes.data), n, cq._ptr(r_h), n, C.byref(rep))
                ctx._check(st, rep.index)

            one()  # this context's workspace
            start.wait()
            for _ in range(ke):
                one()
            start.wait()
            ctx.close() if hasattr(ctx, "close") else None
        except Exception as e:  # pragma: no cover - reported in the line
            errs.append(repr(e))
            start.abort()

    ts = [threading.Thread(target=worker, args=(i,)) for i in range(2)]
    for t in ts:
        t.start()
    try:
        start.wait()
        t0 = time.perf_counter()
        start.wait()
        dt = time.perf_counter() - t0
    except threading.BrokenBarrierError:
        dt = None
    for t in ts:
        t.join()
    if errs or dt is None:
        return {"error": errs[:1]}
    per = dt / (2 * ke)
    return {"value": flops / per / 1e12, "unit": "TFLOP/s", "ms_per_step": per * 1e3, "calls": 2 * ke,
            "note": "two host threads x blocking cqr_factor on two contexts; H2D of one call overlaps D2H of the other"}


def compare_methods(ctx, a, m_global, row0, n, args, stream, dev, world, rdev=None):
    """BASELINE.json configs[1]: CholeskyQR2 and shifted CholeskyQR3 (fixed shift 1e-15,
    experiments.hpp:52) on the same A. CholeskyQR2 breaks down at cond 1e14 (its time is
    the time to the breakdown verdict)."""
    import torch
    import torch.distributed as td

    from paper_2111_11148_b200 import _abi
    from paper_2111_11148_b200 import cholqr as cq
    from paper_2111_11148_b200 import dist

    out = {}
    fixed = _abi.options(shift_kind=_abi.SHIFT_FIXED, shift_value=1e-15)
    q = torch.empty_like(a)
    for name, meth in (("cholqr2", _abi.CHOLQR2), ("scholqr3", _abi.SCHOLQR3)):
        status, pivot = "ok", None

        def one():
            nonlocal status, pivot
            try:
                dist.factor_sharded(ctx, meth, a, m_global, row0, None, fixed, q_out=q)
            except cq.CholeskyBreakdown as e:
                status, pivot = "breakdown", e.pivot_index

        one()
        k = max(3, min(args.steps, 10))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if world > 1:
            td.barrier()
        torch.cuda.synchronize(dev)
        e0.record(stream)
        for _ in range(k):
            one()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        t = torch.tensor([e0.elapsed_time(e1) / k], device=rdev or dev, dtype=torch.float64)
        if world > 1:
            td.all_reduce(t, op=td.ReduceOp.MAX)
        ms = float(t.item())
        d = {"status": status, "ms_per_factorization": ms, "shift": "fixed 1e-15"}
        if status == "ok":
            d["tflops"] = flops_cholqr_family(name, m_global, n) / (ms * 1e-3) / 1e12
            _, r, _ = dist.factor_sharded(ctx, meth, a, m_global, row0, None, fixed, q_out=q)
            d["orth"] = cq.orthogonality_error_dev(q, ctx)
            d["res"] = cq.residual_error_dev(a, q, r, ctx)
        else:
            d["pivot_index"] = pivot
        out[name] = d
    return out


def cpu_baseline(a_dev, m, n, l, method, mname):
    """The oracle (CPU port of the reference) on the SAME A bytes as the GPU arm, the
    whole c1 shape: serial Gaussian sketch as sketch.cpp:94-116, Gram and trisolves on
    all host cores as parexec's workers."""
    import numpy as np

    from oracle import oracle as o
    from paper_2111_11148_b200 import _abi

    a = np.ascontiguousarray(a_dev.cpu().numpy())
    cores = os.cpu_count() or 1
    cfg = _abi.sketch_cfg(strategy=_abi.GAUSSIAN, size=l, rate=RATE, seed=o.derive(SEED, 0x5E7C))
    o.set_test_threads(1)
    t0 = time.perf_counter()
    f = o.factor(method, a, cfg, _abi.options(), workers=cores)
    dt = time.perf_counter() - t0
    stage_s = {nm: f.report.stage_ms[i] / 1e3 for i, nm in enumerate(_abi.STAGE_NAMES) if f.report.stage_ms[i] > 0}
    return {"value": flops_factorization(mname, m, n, l) / dt / 1e12, "unit": "TFLOP/s", "cores": cores,
            "kind": "port", "cpu": cpu_model(), "seconds": dt, "stage_s": stage_s,
            "sample": f"one {mname} factorization of the full c1 A (the GPU arm's bytes, {m} x {n}, l={l}); "
                      f"sketch serial as sketch.cpp:94-116, Gram/trisolves on {cores} workers"}


def run_reference(args):
    """--impl reference: the oracle port on the host cores, rank 0 only."""
    import numpy as np

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import oracle as o
    from paper_2111_11148_b200 import _abi

    mname, _, _, n, l, kap, wdesc = WORKLOADS[args.workload]
    method = {v: k for k, v in _abi.METHOD_NAMES.items()}[mname]
    rows = REF_SAMPLE_ROWS
    # the sample is the first `rows` rows of the reference's own generator applied to the workload's
    # spectrum (matgen.cpp:21-46 restated in the oracle), not our device generator
    a = o.synthesize(rows, n, 1.0, SEED, sigma=workload_sigma(n, kap))
    cores = os.cpu_count() or 1
    cfg = _abi.sketch_cfg(strategy=_abi.GAUSSIAN, size=l, rate=RATE, seed=o.derive(SEED, 0x5E7C))
    o.set_test_threads(1)
    for _ in range(args.warmup):
        o.factor(method, a, cfg, _abi.options(), workers=cores)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        o.factor(method, a, cfg, _abi.options(), workers=cores)
    dt = (time.perf_counter() - t0) / args.steps
    value = flops_factorization(mname, rows, n, l) / dt / 1e12
    line = {"impl": "reference", "metric": METRIC,
            "value": value, "unit": "TFLOP/s", "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": wdesc, "method": mname, "sketch": "gaussian", "n": n, "l": l,
                       "kappa": kap, "sample_rows": rows},
            "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": cores, "kind": "port", "cpu": cpu_model(),
                             "sample": f"{mname} of a {rows} x {n} sample per step (the reference is not buildable "
                                       "here or on the GPU box: no Eigen); serial Gaussian sketch as the reference, "
                                       f"Gram/trisolves on {cores} workers"},
            "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def launch_cmd(argv, gpus):
    """torch.distributed.run command that runs this script once per GPU."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)] + argv


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-compare", action="store_true", help="skip the CholeskyQR2 / sCholeskyQR3 arms (c1)")
    ap.add_argument("--no-overlap", action="store_true", help="skip the two-in-flight e2e extra (c1)")
    ap.add_argument("--dry-run", action="store_true", help="print the multi-GPU launch command and exit")
    ap.add_argument("--transport", default="nccl", choices=["nccl", "host"],
                    help="N > 1: NCCL (one rank per GPU) or the host transport over gloo (ranks may share a GPU)")
    ap.add_argument("--rows", type=int, default=None, help="override the workload's row count (flow checks only)")
    ap.add_argument("--workload", default="c1", choices=sorted(WORKLOADS),
                    help="BASELINE.json config (c1, the benchmark line, by default)")
    args = ap.parse_args(argv)
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    world = os.environ.get("WORLD_SIZE")
    if world is None and args.gpus > 1:
        cmd = launch_cmd(argv, args.gpus)
        if args.dry_run:
            print(json.dumps({"launch": cmd}))
            return 0
        env = dict(os.environ)
        env.setdefault("NCCL_DEBUG", "INFO")
        return subprocess.call(cmd, env=env)
    if world is not None and int(world) != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
    if args.dry_run:
        print(json.dumps({"launch": None, "world": args.gpus}))
        return 0
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)
    return 0


if __name__ == "__main__":
    sys.exit(main())
