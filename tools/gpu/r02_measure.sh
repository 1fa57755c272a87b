# Round-2 measurement set: bench lines of every workload, launch lists, noise sweep
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_c3.json 2> gpurun_out/r02_bench_c3.err; echo c3=$?
for w in c3_cultivation_d3_frame c2_surface_d3_xmem_t c1_surface_d3_zmem c4_color_d5_rz3 c5_surface_d7_r7; do
  timeout 900 python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/r02_bench_$w.json 2> gpurun_out/r02_bench_$w.err; echo $w=$?
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_c3.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-shots 65536 > gpurun_out/r02_launches_c3.log 2>&1; echo launches=$?
timeout 1200 python tools/gpu/noise_sweep.py data/c3_cultivation_d3.zxs.xz 67108864 4096 > gpurun_out/r02_noise_sweep.jsonl 2> gpurun_out/r02_noise_sweep.err; echo sweep=$?
