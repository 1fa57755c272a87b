# A/B (HEAD vs main-lineage speculation), then the dedup parity tests, the cultivation tests and a default bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash tools/gpu/ab_lib.sh data/c3_cultivation_d3.zxs.xz 268435456
rm -rf paper_2604_01059_b200/_lib/ab_*
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "dedup or mono or node or fused or long" > gpurun_out/spec_par.log 2>&1; echo par=$?; tail -2 gpurun_out/spec_par.log
timeout 1500 python -m pytest tests/test_cultivation.py -x -q -m gpu -k "speculation or headline" > gpurun_out/spec_cult.log 2>&1; echo cult=$?; tail -2 gpurun_out/spec_cult.log
ZXS_DEDUP_SPEC=1 timeout 900 python bench.py > gpurun_out/spec_bench.json 2> gpurun_out/spec_bench.err; echo bench=$?; tail -c 1500 gpurun_out/spec_bench.json
