set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -k "long_chain or imag_health" > gpurun_out/pytest30.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest30.log
timeout 900 ncu --section SourceCounters --section WarpStateStats --section InstructionStats --import-source on --clock-control none -k regex:mono_kernel -c 1 -o gpurun_out/prof_mono9t_src30 python tools/gpu/profile_shot.py --model tests/golden/surface_d3_xmem_9t.zxs --shots 3637248 --launches 1 > gpurun_out/ncu30.log 2>&1; echo ncu=$?
tail -2 gpurun_out/ncu30.log
