"""CPU-side checks of the drop-in boundary: the C-ABI library loads without a
GPU, exports every entry point include/cqr.h declares, and its host-only
helpers agree with the oracle (no device work is issued here)."""
import ctypes as C
import os
import re

import pytest

from oracle import oracle as o
from paper_2111_11148_b200 import _abi
from paper_2111_11148_b200 import cholqr as G

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "cqr.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cqr_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(G.LIB_PATH)
    names = declared()
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_abi_struct_sizes_match_header():
    # layout spot checks against the C compiler's view (offsets of trailing fields)
    assert C.sizeof(_abi.SketchCfg) == 56
    assert C.sizeof(_abi.Options) == 32
    assert _abi.Report.sketch_rows.offset > _abi.Report.comm_volume.offset


def test_host_helpers_match_oracle():
    for m, p in [(10, 3), (114, 4), (1000003, 8), (7, 7)]:
        for b in range(p + 1):
            assert G.block_offset(m, p, b) == o.block_offset(m, p, b)
    for meth in (_abi.CHOLQR, _abi.CHOLQR2, _abi.SCHOLQR3, _abi.RLU, _abi.RQR, _abi.RQR_GAUSSIAN):
        assert G.comm_model(meth, 16, 100, 200) == o.comm_model(meth, 16, 100, 200)
    for rate, size in [(0.5, 0), (2.0, 0), (50.0, 0), (2.0, 20)]:
        cfg = G.SketchConfig(rate=rate, size=size)
        assert cfg.resolved_size(100, 10) == o.resolved_size(cfg._c(), 100, 10)


def test_derive_and_orth_names():  # rng.hpp:36-38, apps.cpp:155-162
    for seed, salt in [(0, 0), (1, 0x5E7C), (2**64 - 1, 0xA110 + 3), (123456789, 7)]:
        assert G.derive(seed, salt) == o.derive(seed, salt)
    assert [G.orth_name(x) for x in (G.Orth.HouseholderQr, G.Orth.RqrCholeskyQr, G.Orth.CholeskyQr2)] == \
        ["qr", "rqr", "cholqr2"]


def test_abi_version():
    assert G._lib().cqr_abi_version() == 1


def test_no_cpu_fallback_without_library(monkeypatch, tmp_path):
    monkeypatch.setattr(G, "LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(G, "_LIB", None)
    with pytest.raises(G.DeviceError):
        G.cholesky_qr([[1.0, 0.0], [0.0, 1.0]])
