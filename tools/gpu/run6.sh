set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -x > gpurun_out/pytest_gpu6.log 2>&1; echo pytest=$?
tail -8 gpurun_out/pytest_gpu6.log
timeout 600 python tools/gpu/time_shot.py --model data/c3_cultivation_proxy.zxs.gz --shots 606208 --reps 2 --tag cult_heavy_v2 2>&1 | tee gpurun_out/cult6.json
timeout 300 python tools/gpu/time_shot.py --model tests/golden/surface_d3_xmem_9t.zxs --shots 4194304 --reps 3 --tag 9t_heavy_v2 2>&1 | tee -a gpurun_out/cult6.json
timeout 600 python bench.py --steps 10 --warmup 3 --cpu-seconds 10 > gpurun_out/bench6_c2.json 2>gpurun_out/bench6_c2.err; cat gpurun_out/bench6_c2.json; tail -3 gpurun_out/bench6_c2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches6_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-shots 1048576 > gpurun_out/ncu_launch6.log 2>&1; echo ncul=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:heavy_kernel -s 0 -c 1 -o gpurun_out/prof_heavy_cult6 python tools/gpu/profile_shot.py --model data/c3_cultivation_proxy.zxs.gz --shots 65536 --launches 1 > gpurun_out/ncu6.log 2>&1; echo ncu=$?
tail -3 gpurun_out/ncu6.log
