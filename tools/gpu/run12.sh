set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu12.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_gpu12.log
timeout 300 python tools/gpu/time_shot.py --model tests/golden/surface_d3_xmem_9t.zxs --shots 4194304 --reps 3 --tag 9t_mono_v4 2>&1 | tee gpurun_out/t12.json
timeout 600 python tools/gpu/time_shot.py --model data/c3_cultivation_proxy.zxs.gz --shots 2424832 --reps 2 --tag cult_mono_v4 2>&1 | tee -a gpurun_out/t12.json
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench12_c2.json 2> gpurun_out/bench12_c2.err; echo bench=$?; cat gpurun_out/bench12_c2.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mono_kernel -c 1 -o gpurun_out/prof_mono_9t12 python tools/gpu/profile_shot.py --model tests/golden/surface_d3_xmem_9t.zxs --shots 4194304 --launches 1 > gpurun_out/ncu12a.log 2>&1; echo ncu9t=$?
timeout 900 ncu --section SchedulerStats --section WarpStateStats --section LaunchStats --section Occupancy --section ComputeWorkloadAnalysis --section MemoryWorkloadAnalysis --section SpeedOfLight --clock-control none -k regex:mono_kernel -c 1 -o gpurun_out/prof_mono_cult12 python tools/gpu/profile_shot.py --model data/c3_cultivation_proxy.zxs.gz --shots 2424832 --launches 1 > gpurun_out/ncu12b.log 2>&1; echo ncucult=$?
tail -2 gpurun_out/ncu12a.log gpurun_out/ncu12b.log
