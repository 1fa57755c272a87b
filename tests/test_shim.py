"""The reference-side C++ drop-in (include/zxs_b200_shim.hpp), compiled as a
reference maintainer would (oracle/Makefile `shim`: reference headers and
library + libzxs_b200.so) and run against the reference's own sampler."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "shim_test")


def test_shim_binary_built():
    if not os.path.isdir("/root/reference/proj/include") and not os.path.exists(BIN):
        pytest.skip("reference headers absent and the shim test binary was not shipped")
    assert os.path.exists(BIN), "make -C oracle shim"


@pytest.mark.gpu
@pytest.mark.parametrize("circuit,shots", [("c1_surface_d3_zmem", 100000), ("c2_surface_d3_xmem_t", 65536 + 37)])
def test_shim_matches_reference_sample_detectors(circuit, shots):
    if not os.path.exists(BIN):
        pytest.skip("shim test binary not built")
    out = subprocess.run([BIN, os.path.join(ROOT, "circuits", circuit + ".stim"), str(shots), "3"],
                         capture_output=True, text=True, timeout=600)
    lines = out.stdout.splitlines()
    assert out.returncode == 0, out.stdout + out.stderr
    ok, ones, cached = lines[0].split()
    assert ok == "OK" and int(ones) > 0 and cached == "1"  # second call reused the uploaded sampler
    assert lines[1] == "invalid_argument: sampler was compiled in detector mode"  # sampler.cpp:316-317
