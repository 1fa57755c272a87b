# Round-2 closing set (session 3): spec-kernel A/B, full GPU suite, launch list with DRAM bytes, default bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash tools/gpu/ab_lib.sh data/c3_cultivation_d3.zxs.xz 268435456
rm -rf paper_2604_01059_b200/_lib/ab_*
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/f2_pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/f2_pytest_gpu.log
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/f2_launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-shots 65536 \
  > gpurun_out/f2_launches.log 2>&1; echo launches=$?
timeout 900 python bench.py > gpurun_out/f2_bench.json 2> gpurun_out/f2_bench.err; echo bench=$?; head -c 600 gpurun_out/f2_bench.json
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f2_smoke.log 2>&1; echo smoke=$?; tail -2 gpurun_out/f2_smoke.log
