"""Per-kernel device time of one sample_device call (kernel timing API)."""
import argparse, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import paper_2604_01059_b200 as zx  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="data/c3_cultivation_proxy.zxs.gz")
ap.add_argument("--shots", type=int, default=1 << 24)
ap.add_argument("--tag", default="")
args = ap.parse_args()
cs = zx.CompiledSampler.load(os.path.join(ROOT, args.model))
words = (args.shots + 63) // 64
cols = torch.empty((cs.num_outputs, words), dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream()
for i in range(2):
    cs.sample_device(1, i * args.shots, args.shots, cols.data_ptr(), words, 0, st.cuda_stream)
torch.cuda.synchronize()
cs.kernel_timing(True)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(st)
cs.sample_device(1, 5 * args.shots, args.shots, cols.data_ptr(), words, 0, st.cuda_stream)
b.record(st)
torch.cuda.synchronize()
t = cs.kernel_times()
cs.kernel_timing(False)
print(json.dumps({"tag": args.tag, "shots": args.shots, "total_ms": a.elapsed_time(b), "kernels": t,
                  "info": {k: cs.info[k] for k in ("philox_blocks_per_shot", "num_mono_records", "num_mono_loads")}}))
