set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/gpu/time_shot.py --model data/c3_cultivation_proxy.zxs.gz --shots 606208 --reps 2 --tag cult_heavy_v2 2>&1 | tee gpurun_out/cult7.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:heavy_kernel -s 0 -c 1 -o gpurun_out/prof_heavy_cult7 python tools/gpu/profile_shot.py --model data/c3_cultivation_proxy.zxs.gz --shots 65536 --launches 1 > gpurun_out/ncu7.log 2>&1; echo ncu=$?
tail -3 gpurun_out/ncu7.log
