# ncu of the config-3 (decoded cultivation) deduplicated path at 2^26 shots
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_c3.csv \
  python tools/gpu/load_big.py data/c3_cultivation_d3.zxs.xz 67108864 > gpurun_out/r2_launches_c3.log 2>&1; echo launches=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:dedup_eval_kernel --launch-skip 100 -c 2 \
  -o gpurun_out/r2_ncu_c3_eval python tools/gpu/load_big.py data/c3_cultivation_d3.zxs.xz 67108864 > gpurun_out/r2_ncu_c3_eval.log 2>&1; echo full=$?
