set -x
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -x > gpurun_out/pytest_gpu5.log 2>&1; echo pytest=$?
tail -8 gpurun_out/pytest_gpu5.log
timeout 600 python tools/gpu/time_shot.py --model data/c3_cultivation_proxy.zxs.gz --shots 1212416 --reps 2 --tag cult_heavy_v2 2>&1 | tee gpurun_out/cult5.json
timeout 300 python tools/gpu/time_shot.py --model tests/golden/surface_d3_xmem_9t.zxs --shots 4194304 --reps 3 --tag 9t_heavy_v2 2>&1 | tee -a gpurun_out/cult5.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:heavy_kernel -s 0 -c 1 -o gpurun_out/prof_heavy_cult python tools/gpu/profile_shot.py --model data/c3_cultivation_proxy.zxs.gz --shots 65536 --launches 1 > gpurun_out/ncu5.log 2>&1; echo ncu=$?
tail -3 gpurun_out/ncu5.log
