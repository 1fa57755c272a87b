cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for w in c2_surface_d3_xmem_t c1_surface_d3_zmem c4_color_d5_rz3 c5_surface_d7_r7; do
timeout 900 python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/bench57_$w.json 2> gpurun_out/bench57_$w.err; echo $w=$?; cut -c1-300 gpurun_out/bench57_$w.json
done
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench57_c3.json 2> gpurun_out/bench57_c3.err; echo c3=$?; cut -c1-700 gpurun_out/bench57_c3.json
