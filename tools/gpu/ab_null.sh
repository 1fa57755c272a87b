cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash tools/gpu/ab_lib.sh data/c3_cultivation_d3.zxs.xz 268435456
rm -rf paper_2604_01059_b200/_lib/ab_*
timeout 1500 python -m pytest tests/test_cultivation.py -x -q -m gpu > gpurun_out/null_cult.log 2>&1; echo cult=$?; tail -3 gpurun_out/null_cult.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "dedup or mono or node" > gpurun_out/null_par.log 2>&1; echo par=$?; tail -3 gpurun_out/null_par.log
