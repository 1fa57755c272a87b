"""Debug: dedup variants vs per-shot vs reference on the config-3 frame model."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_2604_01059_b200 as zx
from oracle import refdriver

path = "tests/golden/c3_cultivation_d3_frame.zxs"
shots = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
seed, first = 9, 1 << 30


def load(**env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return zx.CompiledSampler.load(path)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k)
            else:
                os.environ[k] = v


def run(cs, n=shots, f=first):
    return zx.sample_detectors(cs, n, zx.SamplerOptions(seed=seed, force_dense=True), first_shot=f).columns


base = dict(ZXS_HEAVY_MIN_FACTORS="0", ZXS_MONO="1")
recs = {}
for name, env in [("dedup", dict(ZXS_DEDUP="1")), ("split", dict(ZXS_DEDUP="1", ZXS_DEDUP_MAX_KEYS="3000")),
                  ("sync", dict(ZXS_DEDUP="1", ZXS_DEDUP_SYNC="1")), ("nofused", dict(ZXS_DEDUP="1", ZXS_DEDUP_FUSED="0")),
                  ("mono", dict(ZXS_DEDUP="0")), ("default", {})]:
    cs = load(**base, **env) if name != "default" else load()
    if name == "default":
        print("default info", cs.info)
    recs[name] = run(cs)
    print(name, cs.dedup_stats(), flush=True)
    cs.close()


def diff(a, b):
    x = a ^ b
    return [int(np.unpackbits(x[o].view(np.uint8)).sum()) for o in range(x.shape[0])]


names = list(recs)
for i in range(len(names)):
    for j in range(i + 1, len(names)):
        print(names[i], names[j], diff(recs[names[i]], recs[names[j]]), flush=True)
ref = refdriver.RefModel.load(path)
blk = 1 << 16
want = ref.sample_rb(blk, seed, first_shot=first, threads=os.cpu_count())
for n in names:
    print("ref vs", n, diff(recs[n][:, :blk // 64], want), flush=True)
