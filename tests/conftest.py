import pathlib
import sys

import pytest

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libcbct.so")
    config.addinivalue_line("markers", "slow: long-running parity case")
    _ensure_built()


def _ensure_built():
    """The built libraries are git-ignored: a fresh checkout builds them (nvcc cross-compiles
    sm_100a without a GPU) instead of failing the ABI tests spuriously."""
    import subprocess

    targets = [(ROOT / "paper_2110_13526_b200" / "libcbct.so", ROOT / "paper_2110_13526_b200" / "csrc"),
               (ROOT / "oracle" / "liboracle.so", ROOT / "oracle")]
    for so, src in targets:
        if not so.exists() and (src / "Makefile").exists():
            subprocess.run(["make", "-s", "-C", str(src)], check=False)


@pytest.fixture(scope="session")
def golden():
    from _helpers import load_golden

    return load_golden
