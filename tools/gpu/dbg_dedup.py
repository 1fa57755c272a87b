"""Debug: dedup vs per-shot monomial path vs oracle on a fixture."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2604_01059_b200 as zx
from oracle import coracle
from conftest import golden_path

name = sys.argv[1] if len(sys.argv) > 1 else "c2_surface_d3_xmem_t"
def load(d):
    os.environ.update({"ZXS_HEAVY_MIN_FACTORS": "0", "ZXS_MONO": "1", "ZXS_DEDUP": d})
    return zx.CompiledSampler.load(golden_path(name))
a, b = load("1"), load("0")
orc = coracle.OracleModel.load(golden_path(name))
print("comps", a.components)
def samp(cs, shots, seed, first):
    opt = zx.SamplerOptions(seed=seed, force_dense=True)
    f = zx.sample_detectors if cs.mode == zx.MODE_DETECTORS else zx.sample_measurements
    return f(cs, shots, opt, first_shot=first).columns
for shots, seed, first in ((64, 7, 0), (1000, 7, 12345), (5000, 3, 0)):
    A, B = samp(a, shots, seed, first), samp(b, shots, seed, first)
    O = orc.sample(shots, seed, first)
    da = np.unpackbits((A ^ O).view(np.uint8), axis=1, bitorder="little")[:, :shots].sum(1)
    db = np.unpackbits((B ^ O).view(np.uint8), axis=1, bitorder="little")[:, :shots].sum(1)
    print(shots, seed, first, "dedup mismatching rows", np.nonzero(da)[0].tolist(), da[da > 0].tolist(),
          "per-shot", np.nonzero(db)[0].tolist())
# injected f = 0 and uniforms
shots = 256
f = np.zeros((orc.f_width, (shots + 63) // 64), np.uint64)
u = np.random.default_rng(1).random((orc.num_positions, shots))
A = zx.sample_given_f(a, f, shots, uniforms=u)
B = zx.sample_given_f(b, f, shots, uniforms=u)
O = orc.sample(shots, 0, fcols=f, uniforms=u)
print("given f=0: dedup==oracle", np.array_equal(A, O), "per-shot==oracle", np.array_equal(B, O))
if not np.array_equal(A, O):
    d = np.unpackbits((A ^ O).view(np.uint8), axis=1, bitorder="little")[:, :shots]
    print("rows", np.nonzero(d.sum(1))[0].tolist(), "first shots", np.nonzero(d.any(0))[0][:10].tolist())
    for ci, outs in enumerate(a.components):
        print(ci, outs, [int(d[o].sum()) for o in outs])
import json
g = json.load(open(os.path.join(ROOT, "tests/golden/goldens.json")))
a2 = load("1")
for s in g[name]["samples"]:
    if s["shots"] > 200000:
        continue
    A = samp(a2, s["shots"], s["seed"], s["first_shot"])
    O = orc.sample(s["shots"], s["seed"], s["first_shot"])
    d = np.unpackbits((A ^ O).view(np.uint8), axis=1, bitorder="little")[:, :s["shots"]]
    print("golden seq", s["shots"], s["seed"], s["first_shot"], "mismatch rows", np.nonzero(d.sum(1))[0].tolist(),
          "shots", np.nonzero(d.any(0))[0][:8].tolist())
