"""Parity of the sm_100a path against the reference (run on a B200).

Bit-exact gates (integer/bit work and the reference's FP64 arithmetic order):
  * sampled detector/observable records == the reference's sample_detectors /
    sample_measurements (goldens from the unmodified reference, every fixture,
    up to 1e6 shots, shot ranges starting anywhere incl. across 2^32),
  * f-columns == sample_error_batch,
  * eval_batch values == the reference's, bit for bit (FP64 without FMA),
  * injected noise + injected uniforms: run_batch == oracle,
  * Philox uniforms == reference uniform_at,
  * counts == popcounts of the records; any shard split gives the same bits.
Marginal probabilities: probability_of_at within 1e-12 relative (target in
BASELINE.json is 1e-6).
"""
import hashlib

import numpy as np
import pytest

from conftest import fixture_names, golden_path
from oracle import coracle, refdriver

pytestmark = pytest.mark.gpu

import paper_2604_01059_b200 as zx  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, np.uint64).tobytes()).hexdigest()


_cache = {}


def model(name):
    if name not in _cache:
        _cache[name] = zx.CompiledSampler.load(golden_path(name))
    return _cache[name]


def sample(cs, shots, seed, first_shot=0):
    opt = zx.SamplerOptions(seed=seed, force_dense=True)  # the goldens' options
    f = zx.sample_detectors if cs.mode == zx.MODE_DETECTORS else zx.sample_measurements
    return f(cs, shots, opt, first_shot=first_shot).columns


@pytest.mark.parametrize("name", fixture_names())
def test_records_match_reference_goldens(name, goldens):
    cs = model(name)
    for s in goldens[name]["samples"]:
        cols = sample(cs, s["shots"], s["seed"], s["first_shot"])
        assert sha(cols) == s["sha256"], (name, s)


@pytest.mark.parametrize("name", fixture_names())
def test_error_batch_matches_reference(name, goldens):
    cs = model(name)
    for f in goldens[name]["fcols"]:
        fc = zx.sample_error_batch(cs, f["seed"], f["first_shot"], f["shots"])
        assert sha(fc) == f["sha256"], (name, f)


@pytest.mark.parametrize("name", ["c2_surface_d3_xmem_t", "c4_color_d5_rz3", "surface_d3_xmem_rz5",
                                  "surface_d3_xmem_9t", "oracle_mix_4", "random_02", "h_t_h_m"])
def test_eval_batch_bit_exact(name):
    cs = model(name)
    orc = coracle.OracleModel.load(golden_path(name))
    a = orc.arrays
    rng = np.random.default_rng(17)
    shots = 1000 if name != "surface_d3_xmem_9t" else 200
    for c in range(a["comp_out_begin"].size - 1):
        n = int(a["comp_out_begin"][c + 1] - a["comp_out_begin"][c])
        params = rng.integers(0, 2**63, size=(orc.f_width + n, (shots + 63) // 64), dtype=np.uint64)
        for pos in range(n + 1):
            t = int(a["comp_tensor_begin"][c]) + pos
            v_dev = zx.eval_batch(cs, c, pos, params, shots)
            v_orc, mi = orc.eval_batch(t, params, shots)
            assert np.array_equal(v_dev.values.view(np.uint64), v_orc.view(np.uint64)), (name, c, pos)
            assert v_dev.max_imag_ratio == pytest.approx(mi, rel=1e-12, abs=1e-300)


@pytest.mark.parametrize("name", ["c2_surface_d3_xmem_t", "c4_color_d5_rz3", "surface_d3_xmem_rz5", "random_05"])
def test_injected_noise_and_uniforms(name):
    """Bit-exact under injected noise configurations and uniform draws."""
    cs = model(name)
    orc = coracle.OracleModel.load(golden_path(name))
    rng = np.random.default_rng(23)
    shots = 3000
    f = rng.integers(0, 2**63, size=(orc.f_width, (shots + 63) // 64), dtype=np.uint64)
    f[:, -1] &= np.uint64((1 << (shots & 63)) - 1)
    u = rng.random((orc.num_positions, shots))
    try:
        expect = orc.sample(shots, 0, fcols=f, uniforms=u)
    except RuntimeError:
        with pytest.raises(RuntimeError, match="numeric breakdown"):
            zx.sample_given_f(cs, f, shots, uniforms=u)
        return
    assert np.array_equal(zx.sample_given_f(cs, f, shots, uniforms=u), expect)
    # injected noise with the Philox autoregressive draws
    assert np.array_equal(zx.sample_given_f(cs, f, shots, seed=9, first_shot=77),
                          orc.sample(shots, 9, first_shot=77, fcols=f))


def test_philox_matches_reference(goldens):
    for p in goldens["_philox"]:
        assert zx.philox_uniform(p["seed"], p["stream"], p["index"], 1)[0] == p["u"]
    first = 2**32 - 500
    dev = zx.philox_uniform(12345, 0x80000003, first, 1000)
    ref = np.array([coracle.uniform_at(12345, 0x80000003, first + i) for i in range(1000)])
    assert np.array_equal(dev.view(np.uint64), ref.view(np.uint64))


@pytest.mark.skipif(not refdriver.available(), reason="reference library not present")
@pytest.mark.parametrize("name", ["c2_surface_d3_xmem_t", "c4_color_d5_rz3", "oracle_mix_1", "norm_sum",
                                  "random_02", "random_05"])
def test_probability_of_at(name):
    cs = model(name)
    ref = refdriver.RefModel.load(golden_path(name))
    rng = np.random.default_rng(1)
    for _ in range(20):
        outcome = rng.integers(0, 2, cs.num_outputs).astype(np.uint8)
        f = rng.integers(0, 2, cs.f_width).astype(np.uint8)
        try:
            want = ref.probability_of_at(outcome, f)
        except RuntimeError:
            with pytest.raises(RuntimeError):
                zx.probability_of_at(cs, outcome, f)
            continue
        got = zx.probability_of_at(cs, outcome, f)
        assert got == pytest.approx(want, rel=1e-12, abs=1e-300)


@pytest.mark.skipif(not refdriver.available(), reason="reference library not present")
def test_large_d7_against_reference():
    """Config 5 (d=7, 7 rounds): 2^20 shots from shot 2^32-2^19 vs the reference."""
    cs = model("c5_surface_d7_r7")
    ref = refdriver.RefModel.load(golden_path("c5_surface_d7_r7"))
    first, shots = 2**32 - 2**19, 2**20
    assert np.array_equal(sample(cs, shots, 3, first), ref.sample_rb(shots, 3, first_shot=first))


def test_counts_and_shard_invariance():
    """Full-size properties: any split of the shot range gives the same bits
    and counts add up (the multi-GPU sharding contract)."""
    cs = model("c2_surface_d3_xmem_t")
    shots = 1 << 22
    whole = sample(cs, shots, 5)
    counts = zx.count_outputs(cs, shots, seed=5)
    pc = np.unpackbits(whole.view(np.uint8), axis=1).sum(axis=1)
    assert np.array_equal(counts, pc.astype(np.uint64))
    half = shots // 2
    a = sample(cs, half, 5, 0)
    b = sample(cs, half, 5, half)
    assert np.array_equal(np.concatenate([a, b], axis=1), whole)
    c3 = [zx.count_outputs(cs, n, seed=5, first_shot=f) for f, n in ((0, 1000), (1000, shots - 1000))]
    assert np.array_equal(c3[0] + c3[1], counts)


def test_sample_device_strided_and_counts():
    import torch
    cs = model("c4_color_d5_rz3")
    shots, ld = 100_000, 2000
    cols = torch.zeros((cs.num_outputs, ld), dtype=torch.int64, device="cuda")
    counts = torch.zeros(cs.num_outputs, dtype=torch.int64, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    cs.sample_device(3, 0, shots, cols.data_ptr(), ld, counts.data_ptr(), stream)
    cs.check_errors(stream)
    words = (shots + 63) // 64
    got = cols.cpu().numpy().view(np.uint64)
    assert np.array_equal(got[:, :words], sample(cs, shots, 3))
    assert not got[:, words:].any()
    assert np.array_equal(counts.cpu().numpy().view(np.uint64), zx.count_outputs(cs, shots, seed=3))


def test_mode_mismatch_raises_like_reference():
    with pytest.raises(ValueError, match="sampler was compiled in detector mode"):
        zx.sample_measurements(model("c2_surface_d3_xmem_t"), 10)
    with pytest.raises(ValueError, match="sampler was compiled in measurement mode"):
        zx.sample_detectors(model("h_t_h_m"), 10)


def test_ratio_breakdown_raises_like_reference():
    from paper_2604_01059_b200 import zxs_format
    a = zxs_format.load(golden_path("h_t_h_m"))
    t = int(a["tensor_term_begin"][1])
    a["term_c"][2 * t: 2 * int(a["tensor_term_begin"][2])] *= 10.0  # marginal > normalization
    cs = zx.CompiledSampler(a)
    with pytest.raises(RuntimeError, match="autoregressive ratio outside"):
        zx.sample_measurements(cs, 100, zx.SamplerOptions(seed=1))


def test_empty_and_tiny_ranges():
    cs = model("c2_surface_d3_xmem_t")
    assert sample(cs, 0, 1).shape == (25, 0)
    orc = coracle.OracleModel.load(golden_path("c2_surface_d3_xmem_t"))
    for shots, first in ((1, 0), (31, 5), (33, 2**32 - 7), (64, 64), (65, 1)):
        assert np.array_equal(sample(cs, shots, 4, first), orc.sample(shots, 4, first))


def _heavy_model(name, min_factors="1", mono="0", dedup="1"):
    """Sampler whose components (with >= min_factors factors) all run in
    heavy_kernel (mono="0": exact FP64 path) or on the integer monomial path
    (mono="1", where eligible): deduplicated (dedup="1", zxs_dedup.cuh) or
    per shot in mono_kernel (dedup="0")."""
    import os
    keys = {"ZXS_HEAVY_MIN_FACTORS": min_factors, "ZXS_MONO": mono, "ZXS_DEDUP": dedup}
    old = {k: os.environ.get(k) for k in keys}
    os.environ.update(keys)
    try:
        return zx.CompiledSampler.load(golden_path(name))
    finally:
        for k, v in old.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v


@pytest.mark.parametrize("name", ["c2_surface_d3_xmem_t", "c4_color_d5_rz3", "surface_d3_xmem_rz5",
                                  "surface_d3_xmem_9t", "h_t_h_m", "bell_m", "oracle_mix_4", "random_02",
                                  "random_05", "c5_surface_d7_r7"])
def test_heavy_path_matches_reference_goldens(name, goldens):
    """Large-chi path (chunked TMA streaming, 4096 shots per CTA) forced on
    every component: records still equal the reference's bit for bit."""
    cs = _heavy_model(name)
    for s in goldens[name]["samples"]:
        if s["shots"] > 200000:
            continue
        assert sha(sample(cs, s["shots"], s["seed"], s["first_shot"])) == s["sha256"], (name, s)


def test_heavy_path_injected_and_counts():
    name = "c4_color_d5_rz3"
    cs = _heavy_model(name)
    orc = coracle.OracleModel.load(golden_path(name))
    rng = np.random.default_rng(29)
    shots = 5000
    f = rng.integers(0, 2**63, size=(orc.f_width, (shots + 63) // 64), dtype=np.uint64)
    f[:, -1] &= np.uint64((1 << (shots & 63)) - 1)
    u = rng.random((orc.num_positions, shots))
    assert np.array_equal(zx.sample_given_f(cs, f, shots, uniforms=u), orc.sample(shots, 0, fcols=f, uniforms=u))
    full = sample(cs, 70000, 3, 123)
    pc = np.unpackbits(full.view(np.uint8), axis=1).sum(axis=1).astype(np.uint64)
    assert np.array_equal(zx.count_outputs(cs, 70000, seed=3, first_shot=123), pc)


def _heavy_model_path(path):
    import os
    old = os.environ.get("ZXS_MONO")
    os.environ["ZXS_MONO"] = "0"
    try:
        return zx.CompiledSampler.load(path)
    finally:
        if old is None:
            del os.environ["ZXS_MONO"]
        else:
            os.environ["ZXS_MONO"] = old


def test_cultivation_proxy_against_reference():
    """Config-3 proxy (chi = 46,656, 12.4 M factors): the exact FP64 heavy
    path against the reference sampler itself on the same shots."""
    import os
    path = os.path.join(os.path.dirname(golden_path("x")), "..", "..", "data", "c3_cultivation_proxy.zxs.gz")
    if not os.path.exists(path) or not refdriver.available():
        pytest.skip("cultivation proxy not generated (tools/make_fixtures.py --big)")
    cs = _heavy_model_path(path)
    ref = refdriver.RefModel.load(path)
    shots, first = 640, 1 << 20
    got = sample(cs, shots, 11, first)
    want = ref.sample_rb(shots, 11, first_shot=first, batch_size=64, threads=os.cpu_count())
    assert np.array_equal(got, want)


# ---------------------------------------------------------------- monomial path
# surface_d5_r5_xmem_rz3: f_width 122, so its magic component (raw width 125) runs through a
# component-local parameter map (encode_mono)
MONO_NAMES = ["c2_surface_d3_xmem_t", "c4_color_d5_rz3", "surface_d3_xmem_rz5", "surface_d3_xmem_9t", "h_t_h_m",
              "oracle_mix_4", "random_02", "random_05", "steane_inject", "c1_surface_d3_zmem",
              "surface_d5_r5_xmem_rz3"]


@pytest.mark.parametrize("name", MONO_NAMES)
def test_mono_eval_matches_reference(name):
    """Integer monomial contraction vs the reference's eval_batch: relative
    1e-12 of the term-magnitude sum (the reference rounds its h entries)."""
    from test_mono_layout import pack, term_scale
    cs = _heavy_model(name, min_factors="0", mono="1")
    assert cs.info["num_mono_components"] > 0
    orc = coracle.OracleModel.load(golden_path(name))
    arrays = orc.arrays
    rng = np.random.default_rng(5)
    ctb = arrays["comp_tensor_begin"]
    for ci in range(len(ctb) - 1):
        for pos in range(int(ctb[ci + 1] - ctb[ci])):
            tensor = int(ctb[ci]) + pos
            W = max(int(arrays["tensor_param_width"][tensor]), 1)
            shots = 200
            P = rng.integers(0, 2, (shots, W)).astype(np.int64)
            cols = pack(P)
            try:
                got = zx.eval_batch_mono(cs, ci, pos, cols, shots)
            except NotImplementedError:
                continue
            want, _ = orc.eval_batch(tensor, cols, shots)
            err = np.abs(got - want) / (term_scale(arrays, tensor, P) + 1e-300)
            assert err.max() < 1e-12, (name, ci, pos, float(err.max()))


@pytest.mark.parametrize("dedup", ["1", "0"])
@pytest.mark.parametrize("name", MONO_NAMES)
def test_mono_path_matches_reference_goldens(name, dedup, goldens):
    """Records of the monomial path (deduplicated or per shot) == the
    reference's (bit-exact: a difference could only come from a uniform
    falling between the two ratios, ~1e-16 wide; none occurs in these goldens)."""
    cs = _heavy_model(name, min_factors="0", mono="1", dedup=dedup)
    for s in goldens[name]["samples"]:
        if s["shots"] > 200000:
            continue
        assert sha(sample(cs, s["shots"], s["seed"], s["first_shot"])) == s["sha256"], (name, s)


@pytest.mark.parametrize("dedup", ["1", "0"])
def test_mono_injected_noise_ties_counted(dedup):
    """Injected f and uniforms: mono path vs the C oracle. Mismatching bits
    are allowed only at threshold ties (|u - ratio| < 1e-12 at the first
    differing position of a shot); the count is reported."""
    name = "surface_d3_xmem_9t"
    cs = _heavy_model(name, min_factors="0", mono="1", dedup=dedup)
    orc = coracle.OracleModel.load(golden_path(name))
    rng = np.random.default_rng(31)
    shots = 20000
    f = rng.integers(0, 2**63, size=(orc.f_width, (shots + 63) // 64), dtype=np.uint64)
    f[:, -1] &= np.uint64((1 << (shots & 63)) - 1)
    u = rng.random((orc.num_positions, shots))
    got = zx.sample_given_f(cs, f, shots, uniforms=u)
    want = orc.sample(shots, 0, fcols=f, uniforms=u)
    diff = np.unpackbits((got ^ want).view(np.uint8), axis=1, bitorder="little")[:, :shots]
    ties = int(diff.any(axis=0).sum())
    assert ties == 0, f"{ties} shots differ (threshold ties)"


@pytest.mark.parametrize("dedup", ["1", "0"])
def test_mono_counts_and_shards(dedup):
    name = "c4_color_d5_rz3"
    cs = _heavy_model(name, min_factors="0", mono="1", dedup=dedup)
    full = sample(cs, 70000, 3, 123)
    pc = np.unpackbits(full.view(np.uint8), axis=1).sum(axis=1).astype(np.uint64)
    assert np.array_equal(zx.count_outputs(cs, 70000, seed=3, first_shot=123), pc)
    a = sample(cs, 30016, 3, 123)
    b = sample(cs, 70000 - 30016, 3, 123 + 30016)
    assert np.array_equal(np.concatenate([a, b], axis=1)[:, :full.shape[1]], full)


def _load_env(path, **env):
    import os
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return zx.CompiledSampler.load(path)
    finally:
        for k, v in old.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v


@pytest.mark.parametrize("dedup", ["1", "0"])
def test_cultivation_proxy_mono_against_reference(dedup):
    """Config-3 proxy on the monomial path vs the reference sampler itself."""
    import os
    path = os.path.join(os.path.dirname(golden_path("x")), "..", "..", "data", "c3_cultivation_proxy.zxs.gz")
    if not os.path.exists(path) or not refdriver.available():
        pytest.skip("cultivation proxy not generated (tools/make_fixtures.py --big)")
    cs = _load_env(path, ZXS_DEDUP=dedup)
    assert cs.info["num_mono_components"] == 1
    ref = refdriver.RefModel.load(path)
    shots, first = 640, 1 << 20
    got = sample(cs, shots, 11, first)
    want = ref.sample_rb(shots, 11, first_shot=first, batch_size=64, threads=os.cpu_count())
    assert np.array_equal(got, want)


def test_kernel_timing_counts_launches():
    """zxs_kernel_timing/times: one shot_kernel launch per sample call, plus
    mono_kernel when a component is on the monomial path."""
    cs = model("c2_surface_d3_xmem_t")
    cs.kernel_timing(True)
    sample(cs, 10000, 1)
    sample(cs, 10000, 2)
    t = cs.kernel_times()
    cs.kernel_timing(False)
    assert t["shot_kernel"][1] == 2 and t["shot_kernel"][0] > 0 and t["mono_kernel"][1] == 0
    cm = _heavy_model("surface_d3_xmem_9t", min_factors="0", mono="1", dedup="0")
    cm.kernel_timing(True)
    sample(cm, 5000, 1)
    t = cm.kernel_times()
    cm.kernel_timing(False)
    assert t["shot_kernel"][1] == 1 and t["mono_kernel"][1] == 1 and t["dedup_eval_kernel"][1] == 0
    cd = _heavy_model("surface_d3_xmem_9t", min_factors="0", mono="1", dedup="1")
    sample(cd, 5000, 1)  # the first call also contracts the main lineage (once per sampler)
    cd.kernel_timing(True)
    sample(cd, 5000, 1)
    t = cd.kernel_times()
    cd.kernel_timing(False)
    # one chain of 5 outputs (6 tensors) on node levels: 6 evals; aux = speculation init + 6 folds
    # + tensors 0, 1 (key restriction x 2, gather, key-table clear and reset) + level-0 records and
    # a key-table clear and reset + 4 x (node prep + decide + key-table clear and reset) + 5 passes
    # + 5 x (node-table clear and reset)
    assert t["shot_kernel"][1] == 1 and t["mono_kernel"][1] == 0
    assert t["dedup_eval_kernel"][1] == 6
    assert t["dedup_aux"][1] == 1 + 6 + (2 + 1 + 2) + (1 + 2) + 4 * 4 + 5 + 5 * 2


# ---------------------------------------------------------------- deduplicated path
@pytest.mark.parametrize("name", ["surface_d3_xmem_9t", "surface_d3_xmem_rz5", "c4_color_d5_rz3", "steane_inject",
                                  "surface_d5_r5_xmem_rz3"])
def test_dedup_bit_identical_to_per_shot(name):
    """Deduplicated and per-shot monomial paths compute the same canonical
    segment-ordered sums: identical records for every seed and range, and
    identical counts (random f injected too: many distinct keys)."""
    a = _heavy_model(name, min_factors="0", mono="1", dedup="1")
    b = _heavy_model(name, min_factors="0", mono="1", dedup="0")
    assert a.info["num_mono_components"] > 0
    for shots, seed, first in ((1, 1, 0), (33, 2, 5), (100000, 3, 7), (4097, 4, 2**32 - 9)):
        assert np.array_equal(sample(a, shots, seed, first), sample(b, shots, seed, first)), (shots, seed)
    orc = coracle.OracleModel.load(golden_path(name))
    rng = np.random.default_rng(41)
    shots = 30000
    f = rng.integers(0, 2**63, size=(orc.f_width, (shots + 63) // 64), dtype=np.uint64)
    f[:, -1] &= np.uint64((1 << (shots & 63)) - 1)
    u = rng.random((orc.num_positions, shots))
    assert np.array_equal(zx.sample_given_f(a, f, shots, uniforms=u), zx.sample_given_f(b, f, shots, uniforms=u))
    assert np.array_equal(zx.count_outputs(a, 50000, seed=9), zx.count_outputs(b, 50000, seed=9))


@pytest.mark.parametrize("name", ["surface_d3_xmem_9t", "steane_inject", "surface_d5_r5_xmem_rz3"])
def test_dedup_register_staged_forms_identical(name):
    """Block form values computed from register-staged dictionary entries (the path of
    tensors whose staged entries do not fit shared memory; ZXS_DEDUP_STAGE=0 forces it)
    equal the per-shot path's bit for bit."""
    import os
    os.environ["ZXS_DEDUP_STAGE"] = "0"
    try:
        a = _heavy_model(name, min_factors="0", mono="1", dedup="1")
    finally:
        del os.environ["ZXS_DEDUP_STAGE"]
    b = _heavy_model(name, min_factors="0", mono="1", dedup="0")
    orc = coracle.OracleModel.load(golden_path(name))
    rng = np.random.default_rng(43)
    shots = 20000
    f = rng.integers(0, 2**63, size=(orc.f_width, (shots + 63) // 64), dtype=np.uint64)
    f[:, -1] &= np.uint64((1 << (shots & 63)) - 1)
    u = rng.random((orc.num_positions, shots))
    assert np.array_equal(zx.sample_given_f(a, f, shots, uniforms=u), zx.sample_given_f(b, f, shots, uniforms=u))
    assert np.array_equal(sample(a, 70000, 5, 11), sample(b, 70000, 5, 11))


def test_imag_health_check():
    """SURVEY finding 3: the reference never checks that P is real. Clean
    compiles report rounding-level ratios; a model whose magic component's
    coefficients are rotated by theta reports tan(theta) for that component."""
    clean = zx.imag_health(model("c2_surface_d3_xmem_t"), samples=2048)
    assert clean.max() < 1e-9
    arrays = {k: v.copy() for k, v in zx.CompiledSampler.load(golden_path("c2_surface_d3_xmem_t")).arrays.items()}
    tb, ctb = arrays["tensor_term_begin"], arrays["comp_tensor_begin"]
    c = arrays["term_c"].reshape(-1, 2)
    t0 = int(ctb[0])
    sl = slice(int(tb[t0]), int(tb[t0 + 1]))
    th = 0.3
    re, im = c[sl, 0].copy(), c[sl, 1].copy()
    c[sl, 0] = re * np.cos(th) - im * np.sin(th)  # c -> exp(i th) c on one tensor of component 0
    c[sl, 1] = re * np.sin(th) + im * np.cos(th)
    arrays["term_c"] = c.reshape(-1)
    rotated = zx.imag_health(zx.CompiledSampler(arrays), samples=2048)
    assert abs(rotated[0] - np.tan(th)) < 1e-9 and rotated[1:].max() < 1e-9
    # the same metric as the reference's eval_batch on the same parameters
    orc = coracle.OracleModel.load(golden_path("c2_surface_d3_xmem_t"))
    rng = np.random.default_rng(3)
    cs = model("c2_surface_d3_xmem_t")
    P = rng.integers(0, 2**63, size=(int(orc.arrays["tensor_param_width"][1]), 32), dtype=np.uint64)
    mi_dev = zx.eval_batch(cs, 0, 1, P, 2048).max_imag_ratio
    _, mi_ref = orc.eval_batch(int(orc.arrays["comp_tensor_begin"][0]) + 1, P, 2048)
    assert abs(mi_dev - mi_ref) <= 1e-9 * max(mi_ref, 1e-300)  # hypot may differ in the last ulp


def test_dedup_overflow_falls_back_bit_identical():
    """More distinct keys than the tables hold (ZXS_DEDUP_MAX_KEYS=64): the batch
    goes to mono_kernel; records and counts stay identical."""
    import os
    name = "surface_d3_xmem_9t"
    os.environ["ZXS_DEDUP_MAX_KEYS"] = "64"
    try:
        a = _heavy_model(name, min_factors="0", mono="1", dedup="1")
        orc = coracle.OracleModel.load(golden_path(name))
        rng = np.random.default_rng(43)
        shots = 5000
        f = rng.integers(0, 2**63, size=(orc.f_width, (shots + 63) // 64), dtype=np.uint64)
        f[:, -1] &= np.uint64((1 << (shots & 63)) - 1)
        u = rng.random((orc.num_positions, shots))
        got = zx.sample_given_f(a, f, shots, uniforms=u)
        cnt = zx.count_outputs(a, 20000, seed=5)
        small = sample(a, 3000, 2, 11)  # few keys: stays on the deduplicated path after the overflow
    finally:
        del os.environ["ZXS_DEDUP_MAX_KEYS"]
    b = _heavy_model(name, min_factors="0", mono="1", dedup="0")
    assert np.array_equal(got, zx.sample_given_f(b, f, shots, uniforms=u))
    assert np.array_equal(cnt, zx.count_outputs(b, 20000, seed=5))
    assert np.array_equal(small, sample(b, 3000, 2, 11))


def test_dedup_sync_and_async_paths_identical():
    """Device-side key counts (default) and host round trips (ZXS_DEDUP_SYNC=1) give the
    same records; a batch with more keys than one evaluation round is redone synchronously."""
    import os
    name = "surface_d3_xmem_9t"
    a = _heavy_model(name, min_factors="0", mono="1", dedup="1")
    os.environ["ZXS_DEDUP_SYNC"] = "1"
    try:
        b = _heavy_model(name, min_factors="0", mono="1", dedup="1")
    finally:
        del os.environ["ZXS_DEDUP_SYNC"]
    for shots, seed, first in ((5000, 1, 0), (300000, 2, 77)):
        assert np.array_equal(sample(a, shots, seed, first), sample(b, shots, seed, first))
    orc = coracle.OracleModel.load(golden_path(name))
    rng = np.random.default_rng(47)
    shots = 40000  # random f: ~40000 distinct keys
    f = rng.integers(0, 2**63, size=(orc.f_width, (shots + 63) // 64), dtype=np.uint64)
    f[:, -1] &= np.uint64((1 << (shots & 63)) - 1)
    u = rng.random((orc.num_positions, shots))
    a.dedup_stats(reset=True)
    got = zx.sample_given_f(a, f, shots, uniforms=u)
    assert np.array_equal(got, zx.sample_given_f(b, f, shots, uniforms=u))
    assert np.array_equal(got, orc.sample(shots, 0, fcols=f, uniforms=u))


@pytest.mark.parametrize("name", ["surface_d3_xmem_rz5", "c4_color_d5_rz3", "steane_inject"])
def test_dedup_fused_chain_identical(name):
    """Short chains run fused (every position's keys expanded over the sampled-bit
    patterns, one per-shot kernel for the whole chain): same records and counts as the
    step-by-step chain (ZXS_DEDUP_FUSED=0) and as the oracle under injected noise."""
    import os
    a = _heavy_model(name, min_factors="0", mono="1", dedup="1")
    os.environ["ZXS_DEDUP_FUSED"] = "0"
    try:
        b = _heavy_model(name, min_factors="0", mono="1", dedup="1")
    finally:
        del os.environ["ZXS_DEDUP_FUSED"]
    for shots, seed, first in ((4097, 1, 12345), (200000, 2, 0)):
        assert np.array_equal(sample(a, shots, seed, first), sample(b, shots, seed, first))
    assert np.array_equal(zx.count_outputs(a, 100000, seed=5), zx.count_outputs(b, 100000, seed=5))
    orc = coracle.OracleModel.load(golden_path(name))
    rng = np.random.default_rng(53)
    shots = 6000
    f = rng.integers(0, 2**63, size=(orc.f_width, (shots + 63) // 64), dtype=np.uint64)
    f[:, -1] &= np.uint64((1 << (shots & 63)) - 1)
    u = rng.random((orc.num_positions, shots))
    assert np.array_equal(zx.sample_given_f(a, f, shots, uniforms=u), orc.sample(shots, 0, fcols=f, uniforms=u))


@pytest.mark.parametrize("name", ["c4_color_d5_rz3", "steane_inject"])
def test_dedup_fused_chain_overflow(name):
    """A fused chain whose batch has more distinct keys than the tables hold
    (ZXS_DEDUP_MAX_KEYS=64): the garbage pass before the host's redo stays in
    bounds (no sticky fault) and the records equal the per-shot path's."""
    import os
    os.environ["ZXS_DEDUP_MAX_KEYS"] = "64"
    try:
        a = _heavy_model(name, min_factors="0", mono="1", dedup="1")
        orc = coracle.OracleModel.load(golden_path(name))
        rng = np.random.default_rng(59)
        shots = 20000
        f = rng.integers(0, 2**63, size=(orc.f_width, (shots + 63) // 64), dtype=np.uint64)
        f[:, -1] &= np.uint64((1 << (shots & 63)) - 1)
        u = rng.random((orc.num_positions, shots))
        got = zx.sample_given_f(a, f, shots, uniforms=u)
        rec = sample(a, 50000, 3, 7)
    finally:
        del os.environ["ZXS_DEDUP_MAX_KEYS"]
    assert np.array_equal(got, orc.sample(shots, 0, fcols=f, uniforms=u))
    b = _heavy_model(name, min_factors="0", mono="1", dedup="0")
    assert np.array_equal(rec, sample(b, 50000, 3, 7))


@pytest.mark.skipif(not refdriver.available(), reason="reference library not present")
@pytest.mark.parametrize("name,scale", [("c2_surface_d3_xmem_t", 0.9), ("c4_color_d5_rz3", 0.75)])
def test_joint_table_no_hit_fallback(name, scale, tmp_path):
    """A joint mechanism whose table sums to less than 1: a draw above the
    running sum hits nothing and the reference keeps outcome 0
    (sampler.cpp:283-293). Every joint table of the fixture is scaled by
    `scale`, so the no-hit branch fires for ~(1 - scale) of the draws; the
    device records equal the reference sampler's on the same model."""
    from paper_2604_01059_b200 import zxs_format
    a = zxs_format.load(golden_path(name))
    tb, tab = a["mech_table_begin"], a["table"].copy()
    joint = [m for m in range(len(tb) - 1) if tb[m + 1] > tb[m]]
    assert joint
    for m in joint:
        tab[tb[m]:tb[m + 1]] *= scale
    a["table"] = tab
    path = str(tmp_path / "nohit.zxs")
    zxs_format.save(path, a)
    cs = zx.CompiledSampler.load(path)
    ref = refdriver.RefModel.load(path)
    for shots, seed, first in ((20000, 3, 0), (4097, 5, 2**32 - 64)):
        want = ref.sample_rb(shots, seed, first_shot=first, threads=8)
        assert np.array_equal(sample(cs, shots, seed, first), want)
    f_dev = zx.sample_error_batch(cs, 3, 0, 20000)
    assert np.array_equal(f_dev, ref.sample_error_batch(20000, 3))


def test_dedup_overflow_splits_batch():
    """A batch with more distinct keys at some chain position than the tables
    hold is redone as halves on the deduplicated path (down to 2^20 shots)
    before any per-shot fallback: config 3 (frame readout, circuit-level
    noise) at 2^22 shots with 3,000-key tables; records, counts and dedup
    statistics against the per-shot path."""
    import os
    name = "c3_cultivation_d3_frame"
    os.environ["ZXS_DEDUP_MAX_KEYS"] = "3000"
    try:
        a = _heavy_model(name, min_factors="0", mono="1", dedup="1")
        a.dedup_stats(reset=True)
        got = sample(a, 1 << 22, 9, 1 << 30)
        st = a.dedup_stats()
    finally:
        del os.environ["ZXS_DEDUP_MAX_KEYS"]
    b = _heavy_model(name, min_factors="0", mono="1", dedup="0")
    assert np.array_equal(got, sample(b, 1 << 22, 9, 1 << 30))
    assert st["fallbacks"] >= 1  # split (or per-shot) at least once
