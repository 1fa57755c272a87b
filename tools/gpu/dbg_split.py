"""Debug: the batch-split path (ZXS_DEDUP_MAX_KEYS small) vs the per-shot path."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_2604_01059_b200 as zx

path = "tests/golden/c3_cultivation_d3_frame.zxs"
seed, first = 9, 1 << 30
os.environ.update(ZXS_HEAVY_MIN_FACTORS="0", ZXS_MONO="1", ZXS_DEDUP="0")
mono = zx.CompiledSampler.load(path)
os.environ["ZXS_DEDUP"] = "1"
dd = zx.CompiledSampler.load(path)
for shots, mk in [(1 << 22, "3000"), (1 << 21, "3000"), (1 << 22, "100000"), (3 << 20, "3000")]:
    os.environ["ZXS_DEDUP_MAX_KEYS"] = mk
    dd.dedup_stats(reset=True)
    a = zx.sample_detectors(dd, shots, zx.SamplerOptions(seed=seed, force_dense=True), first_shot=first).columns
    st = dd.dedup_stats()
    del os.environ["ZXS_DEDUP_MAX_KEYS"]
    b = zx.sample_detectors(mono, shots, zx.SamplerOptions(seed=seed, force_dense=True), first_shot=first).columns
    x = a ^ b
    bad = np.nonzero(x.any(axis=0))[0]
    print(shots, mk, st, "diff words", len(bad), bad[:10], (bad[-5:] if len(bad) else ""), flush=True)
    if len(bad):
        w = bad[0]
        print("  outputs differing at first word", np.nonzero(x[:, w])[0], [hex(int(v)) for v in a[:, w]], [hex(int(v)) for v in b[:, w]])
