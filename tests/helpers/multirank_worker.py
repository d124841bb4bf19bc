"""One rank of tests/test_gpu_multirank.py: a process that shares cuda:0 with the
other ranks and exchanges through the library's host transport over gloo
(cqr_attach_host_comm). Reads A and the case list from argv[1], writes its Q
rows, R and report fields to argv[1]/rank<r>.npz."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))


def main():
    import torch
    import torch.distributed as td

    from paper_2111_11148_b200 import _abi
    from paper_2111_11148_b200 import cholqr as cq
    from paper_2111_11148_b200 import dist

    d = sys.argv[1]
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    td.init_process_group("gloo", rank=rank, world_size=world,
                          init_method=f"tcp://127.0.0.1:{os.environ['MASTER_PORT']}")
    spec = json.load(open(os.path.join(d, "cases.json")))
    a_full = np.load(os.path.join(d, "a.npy"), mmap_mode="r")
    m, n = a_full.shape
    row0, rows = dist.shard_rows(m, world, rank)
    if spec.get("uneven"):  # not the standard ceil(b*m/p) blocks: the plain-sum Gram path
        cuts = [0] + [int(m * (b + 1) ** 2 / world ** 2) for b in range(world)]
        row0, rows = cuts[rank], cuts[rank + 1] - cuts[rank]
    ctx = cq.Context(0)
    dist.attach_host_transport(ctx)
    a = torch.as_tensor(np.ascontiguousarray(a_full[row0:row0 + rows]), device="cuda:0")
    out = {"row0": row0, "rows": rows}
    for i, c in enumerate(spec["cases"]):
        cfg = cq.SketchConfig(strategy=c["strategy"], size=c.get("size", 0), seed=c["seed"])
        opts = _abi.options(shift_kind=c.get("shift_kind", _abi.SHIFT_THEORY), shift_value=c.get("shift", 0.0))
        try:
            if c.get("host"):
                q, r, rep = dist.factor_sharded_host(ctx, c["method"], a.cpu().numpy(), m, row0, cfg, opts)
                qd = torch.as_tensor(q, device="cuda:0")
            else:
                qd, r, rep = dist.factor_sharded(ctx, c["method"], a, m, row0, cfg, opts)
                q = qd.cpu().numpy()
            out[f"q{i}"], out[f"r{i}"] = q, r
            out[f"st{i}"] = np.array([0, -1, rep.stages[0].retries, rep.comm_rounds, rep.comm_volume])
            out[f"orth{i}"] = np.array([cq.orthogonality_error_dev(qd, ctx), cq.residual_error_dev(a, qd, r, ctx)])
        except cq.CholeskyBreakdown as e:
            out[f"st{i}"] = np.array([_abi.CHOLESKY_BREAKDOWN, e.pivot_index, 0, 0, 0])
        except cq.SingularTriangular as e:
            out[f"st{i}"] = np.array([_abi.SINGULAR_TRIANGULAR, e.index, 0, 0, 0])
    assert not ctx.transport.errors, ctx.transport.errors
    np.savez(os.path.join(d, f"rank{rank}.npz"), **out)
    td.barrier()
    td.destroy_process_group()


if __name__ == "__main__":
    main()
