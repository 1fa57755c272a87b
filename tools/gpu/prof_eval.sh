# ncu --set full of the config-3 dedup_eval_kernel launches 8 and 13..17 (one evaluation round per
# tensor with a 16 GB partial buffer: the big tensors' launches are among them)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
ZXS_DEDUP_PARTIAL_MB=16384 timeout 1500 ncu --set full --clock-control none --import-source on -k regex:dedup_eval_kernel --launch-skip 13 -c 5 \
  -o gpurun_out/r02f_ncu_eval_big python tools/gpu/load_big.py data/c3_cultivation_d3.zxs.xz 268435456 > gpurun_out/r02f_ncu_eval_big.log 2>&1; echo evalbig=$?
ZXS_DEDUP_PARTIAL_MB=16384 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:dedup_eval_kernel --launch-skip 8 -c 1 \
  -o gpurun_out/r02f_ncu_eval_mid python tools/gpu/load_big.py data/c3_cultivation_d3.zxs.xz 268435456 > gpurun_out/r02f_ncu_eval_mid.log 2>&1; echo evalmid=$?
