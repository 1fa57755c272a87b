set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu33.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu33.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke33.log 2>&1; echo smoke=$?; tail -3 gpurun_out/smoke33.log
for w in c2_surface_d3_xmem_t c1_surface_d3_zmem c4_color_d5_rz3; do
timeout 900 python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/bench33_$w.json 2> gpurun_out/bench33_$w.err; echo bench=$?; cat gpurun_out/bench33_$w.json
done
