# Final round-2 set B: launch list + DRAM bytes of one bench step, noise sweep, compute-sanitizer
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/rB_launches_c3.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-shots 65536 \
  > gpurun_out/rB_launches_c3.log 2>&1; echo launches=$?
timeout 1500 python tools/gpu/noise_sweep.py data/c3_cultivation_d3.zxs.xz 67108864 4096 > gpurun_out/rB_noise_sweep.jsonl 2> gpurun_out/rB_noise_sweep.err; echo sweep=$?
timeout 1200 compute-sanitizer --tool memcheck python tools/gpu/sanitize.py > gpurun_out/rB_memcheck.log 2>&1; echo memcheck=$?
timeout 1200 compute-sanitizer --tool racecheck python tools/gpu/sanitize.py > gpurun_out/rB_racecheck.log 2>&1; echo racecheck=$?
