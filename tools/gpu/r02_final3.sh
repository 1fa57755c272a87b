# Round-2 closing set (session 3, after the certain-level skip): full GPU suite, launch list, default bench, smoke
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/gpu/load_big.py data/c3_cultivation_d3.zxs.xz 268435456 268435456 > gpurun_out/f3_load_big.log 2>&1; echo loadbig=$?; grep "shots 268435456" gpurun_out/f3_load_big.log | tail -1 | cut -c1-400
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/f3_launches.csv python bench.py --steps 2 --warmup 0 --no-cpu-baseline --e2e-shots 65536 \
  > gpurun_out/f3_launches.log 2>&1; echo launches=$?
timeout 900 python bench.py > gpurun_out/f3_bench.json 2> gpurun_out/f3_bench.err; echo bench=$?; head -c 400 gpurun_out/f3_bench.json
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f3_smoke.log 2>&1; echo smoke=$?; tail -2 gpurun_out/f3_smoke.log
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/f3_pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/f3_pytest_gpu.log
