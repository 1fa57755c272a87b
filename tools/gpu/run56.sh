cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu56.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu56.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke56.log 2>&1; echo smoke=$?; tail -2 gpurun_out/smoke56.log
timeout 900 python bench.py > gpurun_out/bench56_default.json 2> gpurun_out/bench56_default.err; echo bench=$?; cat gpurun_out/bench56_default.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench56_ref.json 2> gpurun_out/bench56_ref.err; echo ref=$?; cat gpurun_out/bench56_ref.json
ZXS_DEDUP=0 timeout 900 python bench.py --shots $((148*24576)) --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench56_nodedup.json 2> gpurun_out/bench56_nodedup.err; echo nodedup=$?; cut -c1-400 gpurun_out/bench56_nodedup.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches56_default.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-shots 65536 > gpurun_out/ncu_launch56.log 2>&1; echo ncul=$?
