# noise sweep of the deduplicated path after null-space keys + speculation; ncu of the speculation kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python tools/gpu/noise_sweep.py data/c3_cultivation_d3.zxs.xz 67108864 4096 dedup-only > gpurun_out/s3_noise_sweep.jsonl 2> gpurun_out/s3_noise_sweep.err; echo sweep=$?; cat gpurun_out/s3_noise_sweep.jsonl | cut -c1-200
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dedup_init_spec_kernel -c 1 \
  -o gpurun_out/s3_ncu_spec python tools/gpu/load_big.py data/c3_cultivation_d3.zxs.xz 268435456 > gpurun_out/s3_ncu_spec.log 2>&1; echo spec=$?
