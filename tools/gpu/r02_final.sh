# Final round-2 profile set for the default workload (config 3, decoded): launch list with DRAM
# bytes of one bench step, and ncu --set full captures of the hot kernels
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r02_launches_final.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-shots 65536 \
  > gpurun_out/r02_launches_final.log 2>&1; echo launches=$?
# the largest tensor (15) and a middle one (6): a 16 GB partial buffer makes one evaluation round per tensor
ZXS_DEDUP_PARTIAL_MB=16384 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:dedup_eval_kernel --launch-skip 15 -c 1 \
  -o gpurun_out/r02f_ncu_eval_t15 python tools/gpu/load_big.py data/c3_cultivation_d3.zxs.xz 268435456 > gpurun_out/r02f_ncu_eval_t15.log 2>&1; echo eval15=$?
ZXS_DEDUP_PARTIAL_MB=16384 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:dedup_eval_kernel --launch-skip 6 -c 1 \
  -o gpurun_out/r02f_ncu_eval_t6 python tools/gpu/load_big.py data/c3_cultivation_d3.zxs.xz 268435456 > gpurun_out/r02f_ncu_eval_t6.log 2>&1; echo eval6=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"shot_kernel|dedup_node_pass_kernel" -c 3 \
  -o gpurun_out/r02f_ncu_shot_pass python tools/gpu/load_big.py data/c3_cultivation_d3.zxs.xz 268435456 > gpurun_out/r02f_ncu_shot_pass.log 2>&1; echo shotpass=$?
