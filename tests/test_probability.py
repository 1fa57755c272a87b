"""probability_of (sampler.hpp:64, sampler.cpp:370-429) on the device vs the
reference itself: same entropy guard, same DFS enumeration and Kahan sum,
every leaf's outcome_probability_given evaluated on the GPU in the exact FP64
order -> equal bit for bit."""
import itertools
import os
import tempfile

import numpy as np
import pytest

from conftest import golden_path
from oracle import refdriver

pytestmark = pytest.mark.gpu

import paper_2604_01059_b200 as zx  # noqa: E402

# small circuits with 8-18 bits of noise entropy (magic + joint channels)
CIRCUITS = {
    "inject_rep3": """RX 2
T 2
R 0 1 3
CX 2 0 2 1
X_ERROR(0.05) 0 1 2
DEPOLARIZE1(0.02) 3
CX 0 3 1 3
DEPOLARIZE2(0.01) 0 3
M 3
DETECTOR rec[-1]
MX 0 1 2
OBSERVABLE_INCLUDE(0) rec[-1] rec[-2] rec[-3]
DETECTOR rec[-2] rec[-3]
""",
    "rz_noisy": """RX 0 1
R_Z(0.3) 0
T 1
CX 0 2 1 2
X_ERROR(0.1) 0 1 2
Z_ERROR(0.07) 0 1
DEPOLARIZE2(0.03) 0 1
M 2
DETECTOR rec[-1]
MX 0 1
OBSERVABLE_INCLUDE(0) rec[-1]
OBSERVABLE_INCLUDE(1) rec[-2]
""",
}


def _rep5_rounds(rounds=3, p=0.04):
    """5-qubit repetition code, `rounds` syndrome rounds, X_ERROR on every data
    qubit per round (14 mechanisms after channel merging: ~16k leaves), plus a
    T-injected ancilla measured in X."""
    lines = ["R 0 1 2 3 4 5 6 7 8", "RX 9", "T 9", "CX 9 0"]
    for r in range(rounds):
        lines += [f"X_ERROR({p}) 0 1 2 3 4", "CX 0 5 1 5 1 6 2 6 2 7 3 7 3 8 4 8", "M 5 6 7 8", "R 5 6 7 8"]
        for i in range(4):
            lines.append(f"DETECTOR rec[-{4 - i}]" if r == 0 else f"DETECTOR rec[-{4 - i}] rec[-{8 - i}]")
    lines += ["M 0 1 2 3 4", "MX 9", "OBSERVABLE_INCLUDE(0) rec[-2]", "OBSERVABLE_INCLUDE(1) rec[-1]"]
    return "\n".join(lines) + "\n"


CIRCUITS["rep5_r3"] = _rep5_rounds()


def _compile(text, mode=0):
    if not refdriver.available():
        pytest.skip("reference library not built")
    ref = refdriver.RefModel.compile(text, mode)
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "m.zxs")
        ref.save(path)
        cs = zx.CompiledSampler.load(path)
    return ref, cs


@pytest.mark.parametrize("name", sorted(CIRCUITS))
def test_probability_of_matches_reference(name):
    ref, cs = _compile(CIRCUITS[name])
    if cs.num_outputs <= 6:
        outcomes = list(itertools.product((0, 1), repeat=cs.num_outputs))
    else:
        rng = np.random.default_rng(1)
        outcomes = [tuple([0] * cs.num_outputs)] + [tuple(rng.integers(0, 2, cs.num_outputs)) for _ in range(12)]
    total = 0.0
    for bits in outcomes:
        got = zx.probability_of(cs, bits)
        want = ref.probability_of(bits)
        assert got == want, (name, bits, got, want)
        total += got
    if cs.num_outputs <= 6:
        assert abs(total - 1.0) < 1e-9


@pytest.mark.parametrize("name", ["oracle_mix_1", "oracle_mix_2", "random_05", "random_16", "steane_inject",
                                  "steane_inject_shipped", "bell_m", "h_t_h_m"])
def test_probability_of_fixtures(name):
    if not refdriver.available():
        pytest.skip("reference library not built")
    cs = zx.CompiledSampler.load(golden_path(name))
    ref = refdriver.RefModel.load(golden_path(name))
    for bits in itertools.product((0, 1), repeat=min(cs.num_outputs, 4)):
        bits = list(bits) + [0] * (cs.num_outputs - len(bits))
        assert zx.probability_of(cs, bits) == ref.probability_of(bits), (name, bits)


def test_probability_of_errors_like_reference():
    cs = zx.CompiledSampler.load(golden_path("c1_surface_d3_zmem"))
    with pytest.raises(ValueError, match="entropy guard"):
        zx.probability_of(cs, [0] * cs.num_outputs)
    with pytest.raises(ValueError, match="outcome length"):
        zx.probability_of(cs, [0])
