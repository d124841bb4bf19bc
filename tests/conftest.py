import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def pytest_sessionstart(session):
    """A fresh checkout has no built libraries (they are git-ignored): build them once, as
    __graft_entry__.build() does, instead of failing every test on a missing .so."""
    import shutil
    import subprocess

    lib = os.path.join(ROOT, "paper_2111_11148_b200", "libcqr.so")
    orc = os.path.join(ROOT, "oracle", "build", "libcqr_oracle.so")
    if not os.path.exists(lib) and shutil.which("nvcc") and not os.environ.get("CQR_LIB"):
        subprocess.run(["make", "-s", "-j8", "-C", os.path.join(ROOT, "paper_2111_11148_b200", "csrc")], check=False)
    if not os.path.exists(orc):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=False)


def pytest_collection_modifyitems(config, items):
    # GPU tests fail loudly (not skip) when run with -m gpu on a box without a GPU;
    # nothing to do here, the marker only selects.
    pass
