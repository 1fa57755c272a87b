"""Debug: probability_of / eval on a fixture vs the reference (GPU box)."""
import sys, os, itertools
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_2604_01059_b200 as zx
from oracle import refdriver as R
name = sys.argv[1]
path = f"tests/golden/{name}.zxs"
cs = zx.CompiledSampler.load(path)
ref = R.RefModel.load(path)
print(cs.info)
fw = cs.f_width
n = min(1 << fw, 4096)
rng = np.random.default_rng(1)
P = rng.integers(0, 2, (n, fw + 1)).astype(np.uint64)
P[:, fw] = 0
words = (n + 63) // 64
cols = np.zeros((fw + 1, words), np.uint64)
for b in range(fw + 1):
    for i in range(n):
        if P[i, b]:
            cols[b, i >> 6] |= np.uint64(1) << np.uint64(i & 63)
for pos in range(2):
    want, _ = ref.eval_batch(0, pos, cols, n)
    got = zx.eval_batch(cs, 0, pos, cols, n).values
    print("pos", pos, "eval_batch max abs diff", np.abs(got - want).max(), "min norm", want.min(), got.min())
for bits in ([0], [1]):
    try:
        print(bits, "ref", ref.probability_of(bits), "gpu", zx.probability_of(cs, bits))
    except Exception as e:
        print(bits, "ERR", e)
