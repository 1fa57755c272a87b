"""sample_measurements with long autoregressive chains (SURVEY §8 f3,
sampler.cpp:314-320): a T-injected GHZ state of n qubits measured in mixed
bases compiles to one component with an n-long chain. Records equal the
reference's bit for bit on every path that can hold it: the tabulated chain
(n <= 10), the parameter-space light program, global-memory eval, and the
integer monomial kernel."""
import os
import tempfile

import numpy as np
import pytest

from oracle import refdriver

pytestmark = pytest.mark.gpu

import paper_2604_01059_b200 as zx  # noqa: E402


def ghz(n, p=0.01):
    lines = ["RX 0", "T 0"] + [f"CX {i} {i + 1}" for i in range(n - 1)]
    lines += [f"DEPOLARIZE1({p}) " + " ".join(map(str, range(n))), "H 0 2 4", "M " + " ".join(map(str, range(n)))]
    return "\n".join(lines) + "\n"


def _load(ref, env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        with tempfile.TemporaryDirectory() as d:
            path = os.path.join(d, "m.zxs")
            ref.save(path)
            return zx.CompiledSampler.load(path)
    finally:
        for k, v in old.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v


PATHS = {
    "default": {},
    "no_tab": {"ZXS_TAB": "0"},
    "global_eval": {"ZXS_TAB": "0", "ZXS_LIGHT_PROG": "0"},
    "mono": {"ZXS_HEAVY_MIN_FACTORS": "0", "ZXS_MONO": "1"},
}


@pytest.mark.parametrize("n", [8, 14, 20])
@pytest.mark.parametrize("path", sorted(PATHS))
def test_long_chain_matches_reference(n, path):
    if not refdriver.available():
        pytest.skip("reference library not built")
    ref = refdriver.RefModel.compile(ghz(n), 1)
    assert ref.info["max_chain"] == n
    cs = _load(ref, PATHS[path])
    for seed, shots in ((3, 5000), (11, 4097)):
        got = zx.sample_measurements(cs, shots, zx.SamplerOptions(seed=seed, force_dense=True)).columns
        want = ref.sample(shots, seed, force_dense=True)
        assert np.array_equal(got, want), (n, path, seed, shots)
