cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for w in c3_cultivation_proxy c2_surface_d3_xmem_t; do
timeout 900 ncu --set full --clock-control none -k regex:shot_kernel -s 3 -c 1 -o gpurun_out/ncu_full67_$w python bench.py --workload $w --steps 1 --warmup 3 --no-cpu-baseline --e2e-shots 65536 > gpurun_out/ncu67_$w.log 2>&1; echo $w=$?
done
