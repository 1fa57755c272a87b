import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
os.environ["ZXS_HEAVY_MIN_FACTORS"] = "1"
import paper_2604_01059_b200 as zx
from test_mono_layout import pack
name = sys.argv[1] if len(sys.argv) > 1 else "c2_surface_d3_xmem_t"
cs = zx.CompiledSampler.load(os.path.join(ROOT, "tests", "golden", name + ".zxs"))
print(cs.info)
a = cs.arrays
ctb = a["comp_tensor_begin"]
rng = np.random.default_rng(5)
for ci in range(len(ctb) - 1):
    for pos in range(int(ctb[ci + 1] - ctb[ci])):
        t = int(ctb[ci]) + pos
        W = max(int(a["tensor_param_width"][t]), 1)
        P = rng.integers(0, 2, (200, W)).astype(np.int64)
        try:
            v = zx.eval_batch_mono(cs, ci, pos, pack(P), 200)
            print(ci, pos, v[:4])
        except NotImplementedError as e:
            print(ci, pos, "not mono")
