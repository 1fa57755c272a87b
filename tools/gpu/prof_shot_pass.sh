# ncu --set full of the config-3 shot_kernel (one 2^28-shot batch) and two node passes
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:shot_kernel -c 1 \
  -o gpurun_out/r02s_ncu_shot python tools/gpu/load_big.py data/c3_cultivation_d3.zxs.xz 268435456 > gpurun_out/r02s_ncu_shot.log 2>&1; echo shot=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dedup_node_pass_kernel --launch-skip 5 -c 2 \
  -o gpurun_out/r02s_ncu_pass python tools/gpu/load_big.py data/c3_cultivation_d3.zxs.xz 268435456 > gpurun_out/r02s_ncu_pass.log 2>&1; echo pass=$?
