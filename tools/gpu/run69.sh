cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu69.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu69.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke69.log 2>&1; echo smoke=$?; cat gpurun_out/smoke69.log
timeout 900 python bench.py > gpurun_out/bench69_default.json 2> gpurun_out/bench69_default.err; echo bench=$?; cut -c1-600 gpurun_out/bench69_default.json
for s in 1048576 16777216 268435456; do python tools/gpu/dedup_breakdown.py --shots $s --tag size$s 2>&1 | tail -1 | cut -c1-200; done
