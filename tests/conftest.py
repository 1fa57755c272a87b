import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
GOLDEN = os.path.join(ROOT, "tests", "golden")
REFERENCE = "/root/reference/proj"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


def _ensure_built():
    """Builds the checkers and the product library if they are missing
    (build() normally did this already; nvcc cross-compiles without a GPU)."""
    from oracle import coracle, refdriver
    if not coracle.available():
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), os.path.join(ROOT, "oracle", "_ref",
                        "libzxs_oracle.so")], check=True, capture_output=True)
    if not refdriver.available() and os.path.isdir(REFERENCE):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True, capture_output=True)
    from paper_2604_01059_b200 import _native
    if not os.path.exists(_native.LIB_PATH):
        subprocess.run(["make", "-C", os.path.join(ROOT, "paper_2604_01059_b200", "csrc")], check=True,
                       capture_output=True)


_ensure_built()


@pytest.fixture(scope="session")
def goldens():
    with open(os.path.join(GOLDEN, "goldens.json")) as fp:
        return json.load(fp)


def golden_path(name: str) -> str:
    return os.path.join(GOLDEN, name + ".zxs")


def fixture_names():
    with open(os.path.join(GOLDEN, "goldens.json")) as fp:
        return sorted(k for k in json.load(fp) if not k.startswith("_"))


def has_cuda() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
