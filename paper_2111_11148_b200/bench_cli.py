"""Benchmark harness with the reference's CLI and CSV schema, on the device path.

Mirrors proj/tools/bench.cpp (subcommands accuracy | runtime | scaling, grid
syntax of grids.cpp:28-82, exit codes 0 success / 2 usage / 3 I/O) and writes
RunRecord rows with the header of experiments.cpp:45-55:

  method,m,n,l,p,kappa,seed,status,orth_err,res_err,cond_x,t_sketch_ms,...,
  t_householder_ms,t_total_ms,comm_rounds,comm_volume

Inputs come from the device generator (cholqr.synthesize_dev: the reference's
geometric spectrum, seeds derive(seed, 0/1)); the sketch seed is
derive(seed, 0x5E7C) as in experiments.cpp:94; orthogonality and residual are
evaluated on the device (diagnostics.cpp:10-28). Stage times are CUDA-event
milliseconds of the library's stream. `p` is the number of GPUs (ranks under
torchrun; the scaling subcommand reports the current world size).

  python -m paper_2111_11148_b200.bench_cli accuracy --m 100000 --n 100 \
      --kappa 1e3:1e15 --methods rqr,rlu,scholqr3 --seeds 3 --out acc.csv
"""
import argparse
import csv
import math
import os
import sys

from . import _abi
from . import cholqr as cq

STAGES = _abi.STAGE_NAMES
HEADER = (["method", "m", "n", "l", "p", "kappa", "seed", "status", "orth_err", "res_err", "cond_x"] +
          [f"t_{s}_ms" for s in STAGES] + ["t_total_ms", "comm_rounds", "comm_volume"])
METHODS = {v: k for k, v in _abi.METHOD_NAMES.items()}


class UsageError(Exception):
    pass


def parse_grid(text):  # grids.cpp:28-47
    parts = text.split(":")
    if not parts or len(parts) > 3:
        raise UsageError(f"bad grid syntax: '{text}'")
    try:
        vals = [float(p) for p in parts[:2]]
    except ValueError:
        raise UsageError(f"bad number in grid: '{text}'")
    if len(parts) == 1:
        return vals
    lo, hi = vals
    if lo > hi:
        raise UsageError(f"grid lower bound exceeds upper: '{text}'")
    out = []
    if len(parts) == 2 or parts[2] == "log10":
        v = lo
        while v <= hi * (1.0 + 1e-12):
            out.append(v)
            v *= 10.0
    else:
        step = float(parts[2])
        if step <= 0:
            raise UsageError(f"grid step must be positive: '{text}'")
        v = lo
        while v <= hi + step * 1e-9:
            out.append(v)
            v += step
    return out


def parse_methods(text):  # grids.cpp:61-82
    if text == "all":
        return list(range(7))  # grids.cpp:62-66, the HouseholderQr baseline included
    out = []
    for name in text.split(","):
        if name not in METHODS:
            raise UsageError(f"unknown method: '{name}'")
        out.append(METHODS[name])
    if not out:
        raise UsageError("empty method list")
    return out


def parse_shift(text):  # tools/bench.cpp:15-24
    if text == "theory":
        return cq.ShiftMode.theory()
    v = text[6:] if text.startswith("fixed:") else text
    try:
        return cq.ShiftMode.fixed(float(v))
    except ValueError:
        raise UsageError(f"bad --shift-mode: '{text}'")


def fmt(v):
    if v is None:
        return ""
    if isinstance(v, float):
        return repr(v) if math.isfinite(v) else ("inf" if v > 0 else ("-inf" if v < 0 else "nan"))
    return str(v)


def derive(seed, salt):
    m64 = (1 << 64) - 1

    def mix(z):
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m64
        return z ^ (z >> 31)

    return mix(seed ^ mix((salt + 0x51ED270B8A5EC473) & m64))


def measure(ctx, method, a_dev, m, n, kappa, seed, p, cfg, shift, diag, rank_info=None):
    """experiments.cpp:14-43 on the device."""
    import torch

    from . import dist

    sk = cfg
    rec = {"method": _abi.METHOD_NAMES[method], "m": m, "n": n, "p": p, "kappa": kappa, "seed": seed}
    sketched = method in (_abi.RLU, _abi.RQR, _abi.RQR_GAUSSIAN)
    rec["l"] = sk.resolved_size(m, n) if sketched else ""
    opts = _abi.options(diag, False, shift.kind, shift.value, p)
    row0, m_local = (0, m) if rank_info is None else rank_info
    q = torch.empty_like(a_dev)
    try:
        q, r, rep = dist.factor_sharded(ctx, method, a_dev, m, row0, sk, opts, q_out=q)
        rec["status"] = "ok"
        if rank_info is None:
            rec["orth_err"] = cq.orthogonality_error_dev(q, ctx)
            rec["res_err"] = cq.residual_error_dev(a_dev, q, r, ctx)
        conds = [rep.stages[i].cond_x for i in range(rep.n_stages) if rep.stages[i].has_cond_x]
        rec["cond_x"] = conds[-1] if conds else None
        for s, name in enumerate(STAGES):
            rec[f"t_{name}_ms"] = rep.stage_ms[s]
        rec["t_total_ms"] = rep.total_ms
        rec["comm_rounds"], rec["comm_volume"] = rep.comm_rounds, rep.comm_volume
    except cq.CholeskyBreakdown:
        rec["status"] = "breakdown"
    except cq.SingularTriangular:
        rec["status"] = "singular"
    return rec


def main(argv=None):
    ap = argparse.ArgumentParser(prog="bench_cli", description="CholeskyQR benchmark harness (B200)")
    sub = ap.add_subparsers(dest="cmd")
    for name, seeds in (("accuracy", 3), ("runtime", 1), ("scaling", 1)):
        sp = sub.add_parser(name)
        sp.add_argument("--m", default="100000")
        sp.add_argument("--n", default="100")
        sp.add_argument("--kappa", default="1e5")
        sp.add_argument("--p", default="1")
        sp.add_argument("--methods", default="all")
        sp.add_argument("--seeds", type=int, default=seeds)
        sp.add_argument("--seed0", type=int, default=1)
        sp.add_argument("--shift-mode", default="fixed:1e-15")
        sp.add_argument("--l", type=int, default=0)
        sp.add_argument("--rate", default="")
        sp.add_argument("--diag", action="store_true")
        sp.add_argument("--out", required=True)
        if name == "scaling":
            sp.add_argument("--mode", default="strong")
    try:
        args = ap.parse_args(argv)
    except SystemExit as e:
        return 0 if e.code == 0 else 2
    if not args.cmd:
        ap.print_usage(sys.stderr)
        return 2
    try:
        import torch
        import torch.distributed as td

        from . import dist

        shift = parse_shift(args.shift_mode)
        methods = parse_methods(args.methods)
        ms = [int(round(v)) for v in parse_grid(args.m)]
        n = int(round(parse_grid(args.n)[0]))
        kappas = parse_grid(args.kappa)
        if args.cmd != "accuracy":
            kappas = kappas[:1]
        if args.cmd == "scaling" and args.mode not in ("strong", "weak"):
            raise UsageError("--mode must be strong or weak")
        world = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        local = int(os.environ.get("LOCAL_RANK", "0"))
        if world > 1 and not td.is_initialized():
            torch.cuda.set_device(local)
            td.init_process_group("nccl", device_id=torch.device("cuda", local))
        ctx = dist.make_context(local, rank, world)
        records = []
        for m_arg in (ms if args.cmd == "runtime" else ms[:1]):
            m = m_arg * world if (args.cmd == "scaling" and args.mode == "weak") else m_arg
            row0, rows = dist.shard_rows(m, world, rank)
            for kappa in kappas:
                for s in range(args.seeds):
                    seed = args.seed0 + s
                    a = cq.synthesize_dev(rows, n, kappa, seed, device=local, m_global=m, row0=row0, ctx=ctx)
                    for meth in methods:
                        cfg = cq.SketchConfig(size=args.l, rate=float(args.rate) if args.rate else 2.0,
                                              seed=derive(seed, 0x5E7C))
                        rec = measure(ctx, meth, a, m, n, kappa, seed, world, cfg, shift, args.diag,
                                      None if world == 1 else (row0, rows))
                        records.append(rec)
        if rank == 0:
            try:
                with open(args.out, "w", newline="") as f:
                    w = csv.writer(f)
                    w.writerow(HEADER)
                    for r in records:
                        w.writerow([fmt(r.get(h)) for h in HEADER])
            except OSError as e:
                print(f"bench_cli: {e}", file=sys.stderr)
                return 3
        return 0
    except UsageError as e:
        print(f"bench_cli: {e}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
