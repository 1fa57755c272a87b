cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu85.log 2>&1; echo pytest=$?
tail -1 gpurun_out/pytest_gpu85.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke85.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/bench85_c3.json 2> gpurun_out/bench85_c3.err; echo c3=$?; cut -c1-200 gpurun_out/bench85_c3.json
for w in c2_surface_d3_xmem_t c1_surface_d3_zmem c4_color_d5_rz3 c5_surface_d7_r7; do
timeout 900 python bench.py --workload $w > gpurun_out/bench85_$w.json 2> gpurun_out/bench85_$w.err; echo $w=$?; cut -c1-120 gpurun_out/bench85_$w.json
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches85_default.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-shots 65536 > gpurun_out/ncu_launch85.log 2>&1; echo ncul=$?
