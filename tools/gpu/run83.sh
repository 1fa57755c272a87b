cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu83.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu83.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke83.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/bench83_default.json 2> gpurun_out/bench83_default.err; echo bench=$?; cut -c1-700 gpurun_out/bench83_default.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches83_default.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-shots 65536 > gpurun_out/ncu_launch83.log 2>&1; echo ncul=$?
