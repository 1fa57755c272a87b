set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -k "mono" > gpurun_out/pytest_mono8.log 2>&1; echo pytest_mono=$?
tail -30 gpurun_out/pytest_mono8.log
timeout 300 python tools/gpu/time_shot.py --model tests/golden/surface_d3_xmem_9t.zxs --shots 4194304 --reps 3 --tag 9t_mono 2>&1 | tee gpurun_out/t8.json
ZXS_MONO=0 timeout 300 python tools/gpu/time_shot.py --model tests/golden/surface_d3_xmem_9t.zxs --shots 4194304 --reps 3 --tag 9t_heavy 2>&1 | tee -a gpurun_out/t8.json
timeout 600 python tools/gpu/time_shot.py --model data/c3_cultivation_proxy.zxs.gz --shots 2424832 --reps 2 --tag cult_mono 2>&1 | tee -a gpurun_out/t8.json
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -x > gpurun_out/pytest_gpu8.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu8.log
