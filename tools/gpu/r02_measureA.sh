# Final round-2 set A: GPU tests, smoke, bench lines of every workload
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --timeout 1200 > gpurun_out/rA_pytest_gpu.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rA_smoke.log 2>&1; echo smoke=$?
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/rA_bench_c3.json 2> gpurun_out/rA_bench_c3.err; echo c3=$?
for w in c3_cultivation_d3_frame c2_surface_d3_xmem_t c1_surface_d3_zmem c4_color_d5_rz3 c5_surface_d7_r7; do
  timeout 900 python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/rA_bench_$w.json 2> gpurun_out/rA_bench_$w.err; echo $w=$?
done
