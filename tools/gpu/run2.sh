set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -x > gpurun_out/pytest_gpu2.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_gpu2.log
for w in c2_surface_d3_xmem_t c1_surface_d3_zmem c4_color_d5_rz3 c5_surface_d7_r7; do
  timeout 600 python bench.py --steps 5 --warmup 3 --workload $w --cpu-seconds 5 > gpurun_out/bench2_$w.json 2> gpurun_out/bench2_$w.err; echo bench $w=$?
  cat gpurun_out/bench2_$w.json; tail -3 gpurun_out/bench2_$w.err
done
/tmp/px/philox_peak 2>&1 || (nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/philox_peak tools/micro/philox_peak.cu && /tmp/philox_peak) > gpurun_out/philox_peak.txt 2>&1
cat gpurun_out/philox_peak.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:shot_kernel -s 1 -c 1 -o gpurun_out/prof_shot_c2 python tools/gpu/profile_shot.py --shots 16777216 > gpurun_out/ncu2.log 2>&1; echo ncu=$?
tail -3 gpurun_out/ncu2.log
