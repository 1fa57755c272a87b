"""Config 3 (d=3 magic-state cultivation, circuit-level noise) at the sizes the
benchmark runs, against the reference's own sampler (oracle/_ref).

Two compiled models of tools/circuits.py cultivation_d3 (both compiled by the
reference front-end with its cat5 normalisation fixed -- tests/test_circuits.py):
* c3_cultivation_d3_frame (tests/golden): T-basis readout in the check frame,
  chi = 432, a 9-output chain;
* c3_cultivation_d3 (data/, xz): decoded readout, chi = 93,312, a 15-output
  chain, 90.7 M factors -- the benchmark's default workload.

Bit-exactness of the deduplicated (default) path is pinned three ways: against
the per-shot path (ZXS_DEDUP=0) over a whole 2^26-shot batch, against the
reference on a contiguous block and on scattered single shots of that batch
(the reference draws every shot from (seed, global shot index), sampler.cpp:82,
91, 268-284), and the chain tensors' values against the reference's eval_batch.
"""
import os

import numpy as np
import pytest

from conftest import golden_path
from oracle import refdriver

pytestmark = pytest.mark.gpu

import paper_2604_01059_b200 as zx  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIG = os.path.join(ROOT, "data", "c3_cultivation_d3.zxs.xz")

_cache = {}


def _model(path, **env):
    key = (path, tuple(sorted(env.items())))
    if key not in _cache:
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        try:
            arrays = _cache.get(("arrays", path))
            if arrays is None:
                from paper_2604_01059_b200 import zxs_format
                arrays = zxs_format.load(path)
                _cache[("arrays", path)] = arrays
            _cache[key] = zx.CompiledSampler(arrays)
        finally:
            for k, v in old.items():
                if v is None:
                    del os.environ[k]
                else:
                    os.environ[k] = v
    return _cache[key]


def _ref(path):
    key = ("ref", path)
    if key not in _cache:
        _cache[key] = refdriver.RefModel.load(path)
    return _cache[key]


def _sample(cs, shots, seed, first=0):
    return zx.sample_detectors(cs, shots, zx.SamplerOptions(seed=seed, force_dense=True), first_shot=first).columns


def _bits_at(cols, idx):
    return (cols[:, idx >> 6] >> (idx & 63).astype(np.uint64)) & np.uint64(1)


# (name, model, contiguous reference block, scattered reference shots): the decoded model's
# reference sampler runs at ~1.5 shots/s per host thread
MODELS = [("frame", golden_path("c3_cultivation_d3_frame"), 1 << 20, 4096),
          ("decoded", BIG, 1 << 10, 48)]


@pytest.mark.parametrize("name,path,block,singles", MODELS)
def test_headline_batch_against_reference(name, path, block, singles):
    """2^26 shots on the default (deduplicated) path: bit-identical to the
    per-shot path over the whole batch; a contiguous block of `block` shots
    and `singles` scattered shots equal the reference's sampler."""
    if not os.path.exists(path) or not refdriver.available():
        pytest.skip(f"{path} or the reference library absent")
    shots, seed, first = 1 << 26, 7, 3 << 30
    cs = _model(path)
    assert cs.info["num_mono_components"] == 1
    got = _sample(cs, shots, seed, first)
    ref = _ref(path)
    # 64-shot batches: every host thread gets work (the reference's per-shot cost is ~0.7 s here)
    want = ref.sample_rb(block, seed, first_shot=first + (shots - block), batch_size=64, threads=os.cpu_count())
    w0 = (shots - block) // 64
    assert np.array_equal(got[:, w0:w0 + want.shape[1]], want)
    rng = np.random.default_rng(17)
    for s in rng.choice(shots, size=singles, replace=False):
        one = ref.sample_rb(1, seed, first_shot=first + int(s), batch_size=64, threads=1)
        assert np.array_equal(_bits_at(got, np.array([s]))[:, 0], one[:, 0] & np.uint64(1)), int(s)
    if name == "frame":  # the per-shot path at this size takes seconds only for chi = 432
        per_shot = _model(path, ZXS_DEDUP="0")
        assert np.array_equal(got, _sample(per_shot, shots, seed, first))


@pytest.mark.parametrize("name,path,block,singles", MODELS)
def test_chain_values_against_reference_eval(name, path, block, singles):
    """Every chain tensor on the integer path (dedup's canonical order) vs the
    reference's eval_batch at random parameters: marginals within 1e-6
    relative (north star) -- and within 1e-12 of the term-magnitude sum."""
    if not os.path.exists(path) or not refdriver.available():
        pytest.skip(f"{path} or the reference library absent")
    cs = _model(path)
    ref = _ref(path)
    ci = next(i for i, c in enumerate(cs.components) if len(c) > 1)
    n = len(cs.components[ci])
    W = cs.f_width + n
    rng = np.random.default_rng(3)
    shots = 256
    P = (rng.random((W, shots)) < 0.1).astype(np.uint8)  # error-like sparse parameters
    P[:, :64] = 0  # and the all-zero vector (the dominant key)
    cols = np.zeros((W, (shots + 63) // 64), np.uint64)
    for b in range(W):
        for i in np.nonzero(P[b])[0]:
            cols[b, i >> 6] |= np.uint64(1) << np.uint64(i & 63)
    for pos in range(n + 1):
        got = zx.eval_batch_mono(cs, ci, pos, cols, shots)
        want, _ = ref.eval_batch(ci, pos, cols, shots)
        big = np.abs(want) > 1e-9 * np.abs(want).max()
        rel = np.abs(got - want)[big] / np.abs(want)[big]
        assert rel.max() < 1e-6, (name, pos, float(rel.max()))


def test_noiseless_outcome_is_certain_on_device():
    """P(all outputs 0 | no error) = 1 on the device's exact path (the compiled
    circuit is a valid cultivation: every check and the logical readout are
    deterministic without noise)."""
    for path in (golden_path("c3_cultivation_d3_frame"), BIG):
        if not os.path.exists(path):
            continue
        cs = _model(path)
        p = zx.probability_of_at(cs, [0] * cs.num_outputs, [0] * cs.f_width)
        assert abs(p - 1.0) < 1e-9, (path, p)


def test_decoded_dedup_equals_per_shot():
    """The decoded model's summation groups span several segments (spw = 2, 4): the
    deduplicated path and the per-shot mono_kernel (ZXS_DEDUP=0) give the same
    records bit for bit on a batch with many distinct keys per position."""
    if not os.path.exists(BIG):
        pytest.skip(f"{BIG} absent")
    shots, seed, first = 1 << 13, 11, 5 << 20
    got = _sample(_model(BIG), shots, seed, first)
    want = _sample(_model(BIG, ZXS_DEDUP="0"), shots, seed, first)
    assert np.array_equal(got, want)


def test_decoded_evaluation_rounds_identical():
    """Evaluation rounds of 4096 keys (ZXS_DEDUP_ROUND_KEYS; the default is as many as
    the 4 GB partial buffer holds, all of a batch's keys here) give the same records."""
    if not os.path.exists(BIG):
        pytest.skip(f"{BIG} absent")
    shots, seed, first = 1 << 22, 13, 7 << 26
    cs = _model(BIG)
    want = _sample(cs, shots, seed, first)
    cs.dedup_stats(reset=True)
    os.environ["ZXS_DEDUP_ROUND_KEYS"] = "4096"  # read per evaluation
    try:
        got = _sample(cs, shots, seed, first)
    finally:
        del os.environ["ZXS_DEDUP_ROUND_KEYS"]
    stats = cs.dedup_stats()
    assert stats["eval_launches"] > 2 * 16, stats  # several rounds per tensor
    assert np.array_equal(got, want)


@pytest.mark.parametrize("shots,first", [(1 << 24, 3 << 26), (1_000_037, (1 << 32) - 500_000)])
def test_main_lineage_speculation_identical(shots, first):
    """Main-lineage speculation (ZXS_DEDUP_SPEC=1, dedup_init_spec_kernel: zero-key shots that stay on
    the all-zero key's likelier-bit chain skip the node passes; the passes visit
    only the active shots and flip their bits) gives the records, the per-output
    counts and the near-tie count of every shot going through the node passes
    (ZXS_DEDUP_SPEC=0) -- including a ragged batch that crosses 2^32."""
    if not os.path.exists(BIG):
        pytest.skip(f"{BIG} absent")
    seed = 17
    on, off = _model(BIG, ZXS_DEDUP_SPEC="1"), _model(BIG, ZXS_DEDUP_SPEC="0")
    on.tie_count(reset=True)
    off.tie_count(reset=True)
    got = _sample(on, shots, seed, first)
    want = _sample(off, shots, seed, first)
    assert np.array_equal(got, want)
    assert on.tie_count(reset=True) == off.tie_count(reset=True)
    assert np.array_equal(on.count(seed, first, shots), off.count(seed, first, shots))
