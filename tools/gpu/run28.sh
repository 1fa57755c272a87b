set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -k "mono or cultivation" > gpurun_out/pytest_mono28.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_mono28.log
timeout 600 python tools/gpu/time_shot.py --model data/c3_cultivation_proxy.zxs.gz --shots 3637248 --reps 3 --tag cult_mono_v14_generic 2>&1 | tee -a gpurun_out/t28.json
timeout 300 python tools/gpu/time_shot.py --model tests/golden/surface_d3_xmem_9t.zxs --shots 3637248 --reps 3 --tag 9t_mono_v14_generic 2>&1 | tee -a gpurun_out/t28.json
