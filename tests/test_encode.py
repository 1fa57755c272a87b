"""encode_shots (proj/src/encode.cpp:22-48): the C oracle pinned against the
reference itself (CPU), and the device encoder / fused sample+encode against
the oracle bit for bit (GPU)."""
import numpy as np
import pytest

from conftest import golden_path
from oracle import coracle, refdriver


def _random_record(rng, nout, shots):
    words = (shots + 63) // 64
    cols = rng.integers(0, 2**63, size=(nout, words), dtype=np.uint64) ^ (
        rng.integers(0, 2, size=(nout, words), dtype=np.uint64) << np.uint64(63))
    if shots & 63:
        cols[:, -1] &= np.uint64((1 << (shots & 63)) - 1)
    return cols


@pytest.mark.parametrize("nout,shots", [(1, 1), (7, 65), (25, 1000), (33, 64), (337, 130), (0, 5), (8, 0)])
@pytest.mark.parametrize("fmt", [0, 1])
def test_oracle_encode_matches_reference(nout, shots, fmt):
    if not refdriver.available():
        pytest.skip("reference library not built")
    rng = np.random.default_rng(nout * 1000 + shots)
    cols = _random_record(rng, nout, shots)
    assert coracle.encode(cols, shots, fmt) == refdriver.encode(cols, shots, fmt)


def test_oracle_encode_output_range():
    """first_output / output_count clamp like encode.cpp:23-25 (== encoding the column slice)."""
    if not refdriver.available():
        pytest.skip("reference library not built")
    rng = np.random.default_rng(3)
    cols = _random_record(rng, 25, 300)
    for fmt in (0, 1):
        for first, count in ((0, 24), (24, 1), (24, 100), (3, 9), (25, 4), (0, 0)):
            want = refdriver.encode(cols[first:first + count], 300, fmt) if count and first < 25 else (
                b"\n" * 300 if fmt == 0 else b"")
            assert coracle.encode(cols, 300, fmt, first, count) == want, (fmt, first, count)


@pytest.mark.gpu
@pytest.mark.parametrize("nout,shots", [(1, 1), (7, 65), (25, 1000), (33, 64), (337, 1313), (64, 100000)])
@pytest.mark.parametrize("fmt", [0, 1])
def test_device_encode_matches_oracle(nout, shots, fmt):
    import paper_2604_01059_b200 as zx
    rng = np.random.default_rng(nout + shots)
    cols = _random_record(rng, nout, shots)
    assert zx.encode_shots(cols, shots, fmt) == coracle.encode(cols, shots, fmt)
    if nout > 3:
        assert zx.encode_shots(cols, shots, fmt, 2, nout - 3) == coracle.encode(cols, shots, fmt, 2, nout - 3)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c1_surface_d3_zmem", "c2_surface_d3_xmem_t", "c5_surface_d7_r7", "bell_m"])
def test_sample_encoded_matches_cli_path(name):
    """zxs_sample_encoded == encode_shots(sample_*(...)) as the CLI writes it,
    including --separate-observables ranges (zxsim.cpp:155-160)."""
    import paper_2604_01059_b200 as zx
    cs = zx.CompiledSampler.load(golden_path(name))
    opt = zx.SamplerOptions(seed=5)
    shots = 70001
    f = zx.sample_detectors if cs.mode == zx.MODE_DETECTORS else zx.sample_measurements
    rec = f(cs, shots, opt).columns
    for fmt in (0, 1):
        assert zx.sample_encoded(cs, shots, opt, fmt) == coracle.encode(rec, shots, fmt)
        nd = cs.num_detectors
        assert zx.sample_encoded(cs, shots, opt, fmt, 0, nd) == coracle.encode(rec, shots, fmt, 0, nd)
        assert zx.sample_encoded(cs, shots, opt, fmt, nd, cs.num_observables) == coracle.encode(
            rec, shots, fmt, nd, cs.num_observables)
