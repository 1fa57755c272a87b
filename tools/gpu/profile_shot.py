"""Launches the shot kernel a few times on one workload (for ncu captures)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2604_01059_b200 as zx  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="tests/golden/c2_surface_d3_xmem_t.zxs")
ap.add_argument("--shots", type=int, default=1 << 22)
ap.add_argument("--launches", type=int, default=3)
ap.add_argument("--count", action="store_true")
args = ap.parse_args()
cs = zx.CompiledSampler.load(os.path.join(ROOT, args.model))
words = (args.shots + 63) // 64
cols = None if args.count else torch.empty((cs.num_outputs, words), dtype=torch.int64, device="cuda")
counts = torch.zeros(cs.num_outputs, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for i in range(args.launches):
    cs.sample_device(1, i * args.shots, args.shots, 0 if cols is None else cols.data_ptr(), words,
                     counts.data_ptr() if args.count else 0, st)
torch.cuda.synchronize()
cs.check_errors(st)
print("ok", cs.info)
