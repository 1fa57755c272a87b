"""Device time of the shot kernel (CUDA events) for A/B comparisons of builds."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2604_01059_b200 as zx  # noqa: E402
from paper_2604_01059_b200 import _native  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="tests/golden/c2_surface_d3_xmem_t.zxs")
ap.add_argument("--shots", type=int, default=1 << 24)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--tag", default="")
args = ap.parse_args()
cs = zx.CompiledSampler.load(os.path.join(ROOT, args.model))
words = (args.shots + 63) // 64
cols = torch.empty((cs.num_outputs, words), dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream()
cs.sample_device(1, 0, args.shots, cols.data_ptr(), words, 0, st.cuda_stream)
torch.cuda.synchronize()
ts = []
for i in range(args.reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    cs.sample_device(1, (i + 1) * args.shots, args.shots, cols.data_ptr(), words, 0, st.cuda_stream)
    b.record(st)
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
cs.check_errors(st.cuda_stream)
ms = min(ts)
print(json.dumps({"tag": args.tag, "lib": _native.LIB_PATH, "model": args.model, "shots": args.shots, "ms": ms,
                  "shots_per_s": args.shots / ms * 1e3,
                  "philox_blocks_per_s": args.shots * cs.info["philox_blocks_per_shot"] / ms * 1e3}))
