set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -x > gpurun_out/pytest_gpu25.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu25.log
for lib in . r96; do
for m in tests/golden/c2_surface_d3_xmem_t.zxs tests/golden/c1_surface_d3_zmem.zxs tests/golden/c5_surface_d7_r7.zxs tests/golden/c4_color_d5_rz3.zxs; do
ZXS_B200_LIB=$PWD/paper_2604_01059_b200/_lib/$lib/libzxs_b200.so timeout 300 python tools/gpu/time_shot.py --model $m --shots 67108864 --reps 5 --tag tab_$lib 2>&1 | tee -a gpurun_out/t25.json
done; done
ZXS_TAB=0 timeout 300 python tools/gpu/time_shot.py --model tests/golden/c5_surface_d7_r7.zxs --shots 67108864 --reps 5 --tag notab 2>&1 | tee -a gpurun_out/t25.json
