cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:dedup_eval_kernel --launch-skip 0 -c 1 \
  -o gpurun_out/r2_ncu_c3_eval_t0 python tools/gpu/load_big.py data/c3_cultivation_d3.zxs.xz 67108864 > gpurun_out/r2_ncu_c3_eval_t0.log 2>&1; echo t0=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:dedup_eval_kernel --launch-skip 237 -c 1 \
  -o gpurun_out/r2_ncu_c3_eval_t15 python tools/gpu/load_big.py data/c3_cultivation_d3.zxs.xz 67108864 > gpurun_out/r2_ncu_c3_eval_t15.log 2>&1; echo t15=$?
