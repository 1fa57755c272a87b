"""Samples a large-chi model on the deduplicated path (for ncu captures of dedup_eval_kernel)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_2604_01059_b200 as zx

path = sys.argv[1]
shots = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 24
cs = zx.CompiledSampler.load(path)
print(cs.info, flush=True)
for i in range(2):
    rec = zx.sample_detectors(cs, shots, zx.SamplerOptions(seed=1 + i, force_dense=True))
    print(i, int(np.unpackbits(rec.columns.view(np.uint8)).sum()), cs.dedup_stats(reset=True), flush=True)
