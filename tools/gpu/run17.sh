set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for nw in 2 1; do
ZXS_MONO_WORDS=$nw timeout 600 python tools/gpu/time_shot.py --model data/c3_cultivation_proxy.zxs.gz --shots 3637248 --reps 3 --tag cult_mono_v8_nw${nw}_fullwave 2>&1 | tee -a gpurun_out/t17.json
done
timeout 900 python bench.py --workload c3_cultivation_proxy --steps 5 --warmup 3 --e2e-shots 3637248 > gpurun_out/bench17_c3.json 2> gpurun_out/bench17_c3.err; echo bench=$?; cat gpurun_out/bench17_c3.json
timeout 900 ncu --section SchedulerStats --section WarpStateStats --section LaunchStats --section Occupancy --section ComputeWorkloadAnalysis --section MemoryWorkloadAnalysis --section SpeedOfLight --section InstructionStats --clock-control none -k regex:mono_kernel -c 1 -o gpurun_out/prof_mono_cult17 python tools/gpu/profile_shot.py --model data/c3_cultivation_proxy.zxs.gz --shots 3637248 --launches 1 > gpurun_out/ncu17.log 2>&1; echo ncucult=$?
