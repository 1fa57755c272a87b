# A/B (HEAD vs level-0 key restriction), then the dedup parity tests, the cultivation tests and a default bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash tools/gpu/ab_lib.sh data/c3_cultivation_d3.zxs.xz 268435456
rm -rf paper_2604_01059_b200/_lib/ab_*
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "dedup or mono or node" > gpurun_out/l0_par.log 2>&1; echo par=$?; tail -2 gpurun_out/l0_par.log
timeout 1500 python -m pytest tests/test_cultivation.py -x -q -m gpu > gpurun_out/l0_cult.log 2>&1; echo cult=$?; tail -2 gpurun_out/l0_cult.log
timeout 900 python bench.py > gpurun_out/l0_bench.json 2> gpurun_out/l0_bench.err; echo bench=$?; tail -c 1500 gpurun_out/l0_bench.json
