set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -x > gpurun_out/pytest_gpu3.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_gpu3.log
for lib in r64 . r96; do
  for m in tests/golden/c2_surface_d3_xmem_t.zxs tests/golden/c5_surface_d7_r7.zxs tests/golden/c4_color_d5_rz3.zxs; do
    ZXS_B200_LIB=$PWD/paper_2604_01059_b200/_lib/$lib/libzxs_b200.so timeout 300 python tools/gpu/time_shot.py --model $m --shots 16777216 --tag $lib
  done
done 2>&1 | tee gpurun_out/ab3.jsonl
timeout 900 python tools/gpu/time_shot.py --model data/c3_cultivation_proxy.zxs.gz --shots 131072 --reps 2 --tag cult 2>&1 | tee gpurun_out/cult3.json
timeout 600 python - <<'PY' 2>&1 | tee gpurun_out/cult3_ref.json
import sys, time, json, os
sys.path.insert(0, '.')
from oracle import refdriver as R
m = R.RefModel.load('data/c3_cultivation_proxy.zxs.gz')
n = 256
t = time.time(); m.sample(n, 1, threads=os.cpu_count(), batch_size=64); dt = time.time() - t
n = int(max(256, 10 / dt * n)) // 64 * 64
t = time.time(); m.sample(n, 1, threads=os.cpu_count(), batch_size=64); dt = time.time() - t
print(json.dumps({"ref_cultivation_shots_per_s": n / dt, "shots": n, "threads": os.cpu_count(), "s": dt}))
PY
timeout 600 python bench.py --steps 5 --warmup 3 --cpu-seconds 5 > gpurun_out/bench3_c2.json 2>gpurun_out/bench3_c2.err; cat gpurun_out/bench3_c2.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:shot_kernel -s 1 -c 1 -o gpurun_out/prof_shot_c2_v3 python tools/gpu/profile_shot.py --shots 16777216 > gpurun_out/ncu3.log 2>&1; echo ncu=$?
