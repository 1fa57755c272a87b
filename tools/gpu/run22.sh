set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu22.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu22.log
timeout 600 python tools/gpu/time_shot.py --model data/c3_cultivation_proxy.zxs.gz --shots 3637248 --reps 3 --tag cult_mono_v10_basis 2>&1 | tee -a gpurun_out/t22.json
timeout 300 python tools/gpu/time_shot.py --model tests/golden/surface_d3_xmem_9t.zxs --shots 3637248 --reps 3 --tag 9t_mono_v10_basis 2>&1 | tee -a gpurun_out/t22.json
