"""compute-sanitizer driver: the deduplicated / monomial / fused / overflow
paths on small fixtures (run under --tool memcheck / racecheck / synccheck)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_2604_01059_b200 as zx


def load(name, **env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update({k: str(v) for k, v in env.items()})
    try:
        return zx.CompiledSampler.load(f"tests/golden/{name}.zxs")
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def run(cs, shots, seed=1, first=0):
    rec = zx.sample_detectors(cs, shots, zx.SamplerOptions(seed=seed, force_dense=True), first_shot=first)
    return int(np.unpackbits(rec.columns.view(np.uint8)).sum())


for name in ("surface_d3_xmem_9t", "c4_color_d5_rz3", "surface_d5_r5_xmem_rz3", "steane_inject"):
    for env in ({}, {"ZXS_DEDUP_FUSED": 0}, {"ZXS_DEDUP_MAX_KEYS": 64}, {"ZXS_DEDUP": 0}, {"ZXS_DEDUP_SYNC": 1},
                {"ZXS_DEDUP_STAGE": 0}):
        cs = load(name, ZXS_HEAVY_MIN_FACTORS=0, ZXS_MONO=1, **env)
        print(name, env, run(cs, 40000, 1, 12345), zx.count_outputs(cs, 20000, seed=3).sum(), flush=True)
        cs.close()
cs = load("c2_surface_d3_xmem_t")
print("c2", run(cs, 100000), flush=True)
print("SANITIZE-DRIVER-DONE")
