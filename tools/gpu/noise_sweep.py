"""Noise-rate robustness of the deduplicated path (verdict r01 item 8).

The config-3 model's error model rescaled to p' = r x 1e-3 (tools/noise_scale.py:
first order in p, tensors unchanged), sampled on the deduplicated path and per
shot (ZXS_DEDUP=0). Prints one JSON line per (r, path): shots/s (CUDA events
around the device call), distinct keys contracted, fallbacks, near-tie draws.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2604_01059_b200 as zx  # noqa: E402
from paper_2604_01059_b200 import zxs_format  # noqa: E402
from tools.noise_scale import scale  # noqa: E402

path = sys.argv[1] if len(sys.argv) > 1 else "data/c3_cultivation_d3.zxs.xz"
dedup_shots = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 26
mono_shots = int(sys.argv[3]) if len(sys.argv) > 3 else 1 << 14
paths = ("1",) if len(sys.argv) > 4 and sys.argv[4] == "dedup-only" else ("1", "0")
base = zxs_format.load(path)
dev = torch.device("cuda", 0)
for r in (0.1, 1.0, 3.0, 10.0):
    arrays = scale(base, r)
    for dedup in paths:
        os.environ["ZXS_DEDUP"] = dedup
        cs = zx.CompiledSampler(arrays)
        shots = dedup_shots if dedup == "1" else mono_shots
        words = (shots + 63) // 64
        cols = torch.empty((cs.num_outputs, words), dtype=torch.int64, device=dev)
        counts = torch.zeros(cs.num_outputs, dtype=torch.int64, device=dev)
        st = torch.cuda.current_stream(dev)
        cs.sample_device(1, 0, shots, cols.data_ptr(), words, counts.data_ptr(), st.cuda_stream)  # warm-up
        torch.cuda.synchronize()
        cs.dedup_stats(reset=True)
        cs.tie_count(reset=True)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        cs.sample_device(1, shots, shots, cols.data_ptr(), words, counts.data_ptr(), st.cuda_stream)
        b.record(st)
        torch.cuda.synchronize()
        cs.check_errors(st.cuda_stream)
        ms = a.elapsed_time(b)
        d = cs.dedup_stats()
        print(json.dumps({"noise_scale": r, "p": r * 1e-3, "dedup": dedup == "1", "shots": shots,
                          "shots_per_s": shots / (ms / 1e3), "ms": ms, "keys": d["keys"], "fallbacks": d["fallbacks"],
                          "ties": cs.tie_count(), "ones_per_shot": float(counts.sum().item()) / (2 * shots)}),
              flush=True)
        cs.close()
