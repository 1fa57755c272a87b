set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for k in 100 2 1 0; do
ZXS_DEBUG_AR_COMPONENTS=$k timeout 300 python tools/gpu/time_shot.py --model tests/golden/c2_surface_d3_xmem_t.zxs --shots 67108864 --reps 5 --tag c2_ar$k 2>&1 | tee -a gpurun_out/t24.json
done
ZXS_HEAVY_MIN_FACTORS=0 timeout 300 python tools/gpu/time_shot.py --model tests/golden/c4_color_d5_rz3.zxs --shots 3637248 --reps 3 --tag c4_mono 2>&1 | tee -a gpurun_out/t24.json
timeout 300 python tools/gpu/time_shot.py --model tests/golden/c4_color_d5_rz3.zxs --shots 3637248 --reps 3 --tag c4_light 2>&1 | tee -a gpurun_out/t24.json
