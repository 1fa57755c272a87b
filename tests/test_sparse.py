"""The reference's sparse geometric path (sampler.cpp:104-147, 214-255) on the
device: pure-Clifford deterministic models with single mechanisms (p < 1) and
few expected flips take it by default (SamplerOptions.sparse_threshold = 8,
force_dense = false), exactly as the reference does. Records are compared with
the reference's own sample_detectors bit for bit (its gaps use log/log1p; the
device uses the reference's log1p(-p) and CUDA's log, which could only differ
at a floor boundary -- none occurs here)."""
import os
import tempfile

import numpy as np
import pytest

from oracle import coracle, refdriver


def pair_parity(k=8, p=0.001, extra=""):
    """k qubit pairs with X_ERROR on every qubit, detectors = pair parities
    (plus one cross parity), observable = a two-measurement parity: every
    mechanism a single, no magic, and the reference compiles every output to a
    DirectOutput (single-measurement detectors become autoregressive
    components in this compiler, SURVEY finding 7)."""
    q = " ".join(str(i) for i in range(2 * k))
    t = f"R {q}\nX_ERROR({p}) {q}\n{extra}M {q}\n"
    for i in range(k):
        t += f"DETECTOR rec[-{2 * i + 1}] rec[-{2 * i + 2}]\n"
    t += "DETECTOR rec[-1] rec[-3]\nOBSERVABLE_INCLUDE(0) rec[-2] rec[-4]\n"
    return t


CX_CIRCUIT = """R 0 1 2 3
X_ERROR(0.01) 0 1 2 3
CX 0 1 2 3
X_ERROR(0.03) 1 3
Z_ERROR(0.02) 0
M 0 1 2 3
DETECTOR rec[-1] rec[-2]
DETECTOR rec[-3] rec[-4]
DETECTOR rec[-1] rec[-3]
OBSERVABLE_INCLUDE(0) rec[-2] rec[-4]
"""


def _compile(text):
    if not refdriver.available():
        pytest.skip("reference library not built")
    return refdriver.RefModel.compile(text, 0)


def test_flags_roundtrip_through_zxs():
    """The .zxs header carries stats.pure_clifford_deterministic (compile.cpp:324-325)."""
    from paper_2604_01059_b200 import zxs_format
    ref = _compile(pair_parity())
    assert ref.info["pure_clifford_deterministic"] == 1 and ref.info["num_components"] == 0
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "m.zxs")
        ref.save(path)
        arrays = zxs_format.load(path)
        assert arrays["header"].size == 6 and arrays["header"][5] & 1
        assert zxs_format.make_desc(arrays).flags & 1
        assert refdriver.RefModel.load(path).info["pure_clifford_deterministic"] == 1


@pytest.mark.gpu
@pytest.mark.parametrize("text", [pair_parity(8, 0.001), pair_parity(16, 0.05), pair_parity(4, 0.2), CX_CIRCUIT],
                         ids=["pairs8", "pairs16", "pairs4_p02", "cx"])
def test_sparse_path_matches_reference(text):
    import paper_2604_01059_b200 as zx
    ref = _compile(text)
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "m.zxs")
        ref.save(path)
        cs = zx.CompiledSampler.load(path)
    assert zx.sparse_eligible(cs)
    assert not zx.sparse_eligible(cs, zx.SamplerOptions(force_dense=True))
    for seed, shots in ((1, 1000), (7, 100003), (123, 64), (5, 1)):
        got = zx.sample_detectors(cs, shots, zx.SamplerOptions(seed=seed)).columns
        want = ref.sample(shots, seed, force_dense=False)
        assert np.array_equal(got, want), (seed, shots)
        dense = zx.sample_detectors(cs, shots, zx.SamplerOptions(seed=seed, force_dense=True)).columns
        assert np.array_equal(dense, ref.sample(shots, seed, force_dense=True)), (seed, shots)
    # the CLI write path honours the same options
    shots = 4097
    rec = ref.sample(shots, 3, force_dense=False)
    for fmt in (0, 1):
        assert zx.sample_encoded(cs, shots, zx.SamplerOptions(seed=3), fmt) == coracle.encode(rec, shots, fmt)


@pytest.mark.gpu
def test_sparse_threshold_gates_like_reference():
    import paper_2604_01059_b200 as zx
    ref = _compile(pair_parity(16, 0.4))  # expected flips per shot > 8: dense
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "m.zxs")
        ref.save(path)
        cs = zx.CompiledSampler.load(path)
    assert not zx.sparse_eligible(cs)
    assert zx.sparse_eligible(cs, zx.SamplerOptions(sparse_threshold=1e9))
    got = zx.sample_detectors(cs, 5000, zx.SamplerOptions(seed=2)).columns
    assert np.array_equal(got, ref.sample(5000, 2, force_dense=False))
    got = zx.sample_detectors(cs, 5000, zx.SamplerOptions(seed=2, sparse_threshold=1e9)).columns
    assert np.array_equal(got, ref.sample_opts(5000, 2, sparse_threshold=1e9))
