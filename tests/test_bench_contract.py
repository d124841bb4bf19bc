"""bench.py keeps the driver's JSON-line contract: the reference arm on CPU (the
oracle port on the host cores, runs here), our arm on the B200 (gpu marker)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args, timeout=900):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                         text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config"}


def test_reference_arm_line():
    d = _run("--impl", "reference", "--steps", "1", "--warmup", "1")
    assert BASE_KEYS <= d.keys()
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "TFLOP/s"
    assert d["cpu_baseline"]["kind"] in ("port", "reference") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["config"]["workload"].startswith("c1")


@pytest.mark.gpu
def test_our_arm_line():
    d = _run("--steps", "3", "--warmup", "3", "--no-cpu")
    assert BASE_KEYS <= d.keys()
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
    assert d["dtype"] == "f64" and d["higher_is_better"] is True
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor") and r["frac"] > 0 and r["peak"] > 0
    # The sketch's FP64-equivalent rate is counted against the FP64 (DMMA) roof north_star names, but the exact
    # product runs on the int8 tensor cores: it may pass the DMMA peak, and then the line must also carry the
    # roof of the unit it really runs on, which bounds it.
    assert r["frac"] <= 1 or 0 < r["int8_emulation"]["frac"] <= 1
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert e["two_in_flight"]["value"] > 0  # the extra: two blocking calls in flight from two host threads
    assert d["gpu_launches"] > 0 and "sm_mhz" in d["clocks"]
    assert set(d["stage_roofline"]) >= {"sketch", "gram", "trisolve"}
    assert d["check"]["orth"] < 1e-10


@pytest.mark.gpu
@pytest.mark.parametrize("workload,rows", [("c2", 300_001), ("c1", 150_000)])
def test_n_rank_flow_on_one_gpu(workload, rows):
    """bench.py --gpus 2 end to end (launcher, shards, sharded factorization and e2e, max over ranks, one
    line from rank 0) with the ranks sharing this GPU over the host transport; NCCL needs one GPU per rank."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--transport", "host",
                          "--workload", workload, "--rows", str(rows), "--steps", "2", "--warmup", "3", "--no-cpu"],
                         cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert BASE_KEYS <= d.keys() and d["n_gpus"] == 2 and d["value"] > 0
    weak = workload == "c1"
    assert d["scaling"] == ("weak" if weak else "strong")
    assert d["config"]["m_global"] == (2 * rows if weak else rows)
    assert d["check"]["orth"] < 1e-10 and d["check"]["res"] < 1e-12
    assert d["e2e"]["value"] > 0 and "cqr_factor_sharded" in d["e2e"]["api"]
    assert d["config"]["transport"].startswith("host")


def test_multi_gpu_launcher_dry_run():
    """--gpus N without WORLD_SIZE re-launches under torch.distributed.run, one rank per GPU."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "8", "--workload", "c2",
                          "--dry-run"], cwd=ROOT, capture_output=True, text=True, timeout=120, env=env)
    assert out.returncode == 0, out.stderr
    cmd = json.loads(out.stdout.strip().splitlines()[-1])["launch"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"] and "--nproc-per-node=8" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    i = cmd.index(os.path.join(ROOT, "bench.py"))
    assert cmd[i + 1:i + 5] == ["--gpus", "8", "--workload", "c2"]
    # under the launcher WORLD_SIZE must agree with --gpus
    bad = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "8"], cwd=ROOT,
                         capture_output=True, text=True, timeout=120, env=dict(env, WORLD_SIZE="2"))
    assert bad.returncode == 2


def test_strong_and_weak_shards():
    """c2 is strong-scaled (fixed m = 4e6, ceil(b*m/p) blocks, parexec.cpp:13-15); c1/c3 weak."""
    sys.path.insert(0, ROOT)
    import bench

    for p in (1, 2, 4, 8):
        rows = [bench.workload_shape("c2", p, b) for b in range(p)]
        assert sum(r[3] for r in rows) == 4_000_000 and all(r[1] == 4_000_000 for r in rows)
        assert [r[2] for r in rows] == [-(-b * 4_000_000 // p) for b in range(p)]
        w = [bench.workload_shape("c3", p, b) for b in range(p)]
        assert all(r[3] == 4_194_304 for r in w) and w[0][1] == 4_194_304 * p
    assert bench.shard(10, 3, 0) == (0, 4) and bench.shard(10, 3, 1) == (4, 3) and bench.shard(10, 3, 2) == (7, 3)
