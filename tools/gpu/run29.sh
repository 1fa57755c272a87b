set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu29.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu29.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke29.log 2>&1; echo smoke=$?; cat gpurun_out/smoke29.log
t0=$(date +%s); timeout 900 python bench.py > gpurun_out/bench29_default.json 2> gpurun_out/bench29_default.err; echo bench=$? secs=$(( $(date +%s) - t0 )); cat gpurun_out/bench29_default.json
timeout 900 python bench.py --workload c2_surface_d3_xmem_t --steps 10 --warmup 3 > gpurun_out/bench29_c2.json 2> gpurun_out/bench29_c2.err; echo benchc2=$?; cat gpurun_out/bench29_c2.json
timeout 900 python bench.py --workload c4_color_d5_rz3 --steps 10 --warmup 3 > gpurun_out/bench29_c4.json 2> gpurun_out/bench29_c4.err; echo benchc4=$?
timeout 900 python bench.py --workload c5_surface_d7_r7 --steps 10 --warmup 3 > gpurun_out/bench29_c5.json 2> gpurun_out/bench29_c5.err; echo benchc5=$?
timeout 900 python bench.py --workload c1_surface_d3_zmem --steps 10 --warmup 3 > gpurun_out/bench29_c1.json 2> gpurun_out/bench29_c1.err; echo benchc1=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 24 --csv --log-file gpurun_out/launches29_default.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-shots 65536 > gpurun_out/ncu_launch29.log 2>&1; echo ncul=$?
