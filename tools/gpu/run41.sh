cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu41.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu41.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke41.log 2>&1; echo smoke=$?; tail -2 gpurun_out/smoke41.log
t0=$(date +%s); timeout 900 python bench.py > gpurun_out/bench41_default.json 2> gpurun_out/bench41_default.err; echo bench=$? secs=$(( $(date +%s) - t0 )); cat gpurun_out/bench41_default.json; tail -3 gpurun_out/bench41_default.err
