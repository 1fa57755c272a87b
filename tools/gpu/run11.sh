set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -k "mono" > gpurun_out/pytest_mono11.log 2>&1; echo pytest_mono=$?
tail -4 gpurun_out/pytest_mono11.log
timeout 300 python tools/gpu/time_shot.py --model tests/golden/surface_d3_xmem_9t.zxs --shots 4194304 --reps 3 --tag 9t_mono_v2 2>&1 | tee gpurun_out/t11.json
timeout 600 python tools/gpu/time_shot.py --model data/c3_cultivation_proxy.zxs.gz --shots 2424832 --reps 2 --tag cult_mono_v2 2>&1 | tee -a gpurun_out/t11.json
timeout 900 python bench.py --workload c3_cultivation_proxy --steps 5 --warmup 3 --e2e-shots 2424832 > gpurun_out/bench11_c3.json 2> gpurun_out/bench11_c3.err; echo bench=$?; cat gpurun_out/bench11_c3.json; tail -3 gpurun_out/bench11_c3.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mono_kernel -c 1 -o gpurun_out/prof_mono_cult11 python tools/gpu/profile_shot.py --model data/c3_cultivation_proxy.zxs.gz --shots 2424832 --launches 1 > gpurun_out/ncu11.log 2>&1; echo ncu=$?
tail -3 gpurun_out/ncu11.log
