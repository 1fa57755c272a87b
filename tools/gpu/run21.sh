set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
t0=$(date +%s); timeout 900 python bench.py > gpurun_out/bench21_default.json 2> gpurun_out/bench21_default.err; echo bench=$? secs=$(( $(date +%s) - t0 )); cat gpurun_out/bench21_default.json
t0=$(date +%s); timeout 900 python bench.py --impl reference > gpurun_out/bench21_ref.json 2> gpurun_out/bench21_ref.err; echo ref=$? secs=$(( $(date +%s) - t0 )); cat gpurun_out/bench21_ref.json
timeout 900 ncu --section SourceCounters --section WarpStateStats --section InstructionStats --import-source on --clock-control none -k regex:mono_kernel -c 1 -o gpurun_out/prof_mono_src21 python tools/gpu/profile_shot.py --model data/c3_cultivation_proxy.zxs.gz --shots 3637248 --launches 1 > gpurun_out/ncu21.log 2>&1; echo ncu=$?
