# Round-2 closing set (session 3, last): targeted GPU tests of the speculation path, default bench, launch list, smoke
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "dedup or node or timing or fused" > gpurun_out/f4_par.log 2>&1; echo par=$?; tail -1 gpurun_out/f4_par.log
timeout 1500 python -m pytest tests/test_cultivation.py -q -m gpu -k "speculation or rounds or per_shot" > gpurun_out/f4_cult.log 2>&1; echo cult=$?; tail -1 gpurun_out/f4_cult.log
timeout 900 python bench.py > gpurun_out/f4_bench.json 2> gpurun_out/f4_bench.err; echo bench=$?; head -c 300 gpurun_out/f4_bench.json
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/f4_launches.csv python bench.py --steps 2 --warmup 0 --no-cpu-baseline --e2e-shots 65536 \
  > gpurun_out/f4_launches.log 2>&1; echo launches=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f4_smoke.log 2>&1; echo smoke=$?; tail -2 gpurun_out/f4_smoke.log
