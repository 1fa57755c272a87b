"""Loads a large compiled model and times sampler creation + a few batches (GPU box)."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_2604_01059_b200 as zx
from paper_2604_01059_b200 import zxs_format

path = sys.argv[1]
t = time.time()
arrays = zxs_format.load(path)
print(f"load {time.time() - t:.1f}s", flush=True)
t = time.time()
cs = zx.CompiledSampler(arrays)
print(f"create {time.time() - t:.1f}s", cs.info, flush=True)
for shots in [int(x) for x in sys.argv[2:]] or [1 << 20, 1 << 24]:
    cs.kernel_timing(True)
    cs.dedup_stats(reset=True)
    t = time.time()
    rec = zx.sample_detectors(cs, shots, zx.SamplerOptions(seed=1, force_dense=True))
    dt = time.time() - t
    kt = cs.kernel_times()
    cs.kernel_timing(False)
    print(f"shots {shots}: {dt:.3f}s {shots / dt:.3e} shots/s ones {int(np.unpackbits(rec.columns.view(np.uint8)).sum())}",
          cs.dedup_stats(), {k: (round(v, 2), n) for k, (v, n) in kt.items() if n}, "ties", cs.tie_count(reset=True), flush=True)
