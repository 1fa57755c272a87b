set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu15.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_gpu15.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke15.log 2>&1; echo smoke=$?; cat gpurun_out/smoke15.log
timeout 900 python bench.py --workload c3_cultivation_proxy --steps 5 --warmup 3 --e2e-shots 2424832 > gpurun_out/bench15_c3.json 2> gpurun_out/bench15_c3.err; echo bench=$?; cat gpurun_out/bench15_c3.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 20 --csv --log-file gpurun_out/launches15_c3.csv python bench.py --workload c3_cultivation_proxy --steps 2 --warmup 3 --no-cpu-baseline --e2e-shots 65536 > gpurun_out/ncu_launch15.log 2>&1; echo ncul=$?
