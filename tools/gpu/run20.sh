set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -x > gpurun_out/pytest_gpu20.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu20.log
for lp in 1 0; do
for m in tests/golden/c2_surface_d3_xmem_t.zxs tests/golden/c1_surface_d3_zmem.zxs tests/golden/c4_color_d5_rz3.zxs; do
ZXS_LIGHT_PROG=$lp timeout 300 python tools/gpu/time_shot.py --model $m --shots 16777216 --reps 5 --tag light$lp 2>&1 | tee -a gpurun_out/t20.json
done; done
