# A/B of the summation-segment cap on config 3 (decoded), 2^28 shots per batch
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for g in 2368 1184 592 296; do
  ZXS_DEDUP_SEGS=$g timeout 600 python tools/gpu/load_big.py data/c3_cultivation_d3.zxs.xz 268435456 268435456 > gpurun_out/r2_ab_segs_$g.log 2>&1
  echo "segs=$g"; grep "shots 268435456" gpurun_out/r2_ab_segs_$g.log | tail -1 | cut -c1-400
done
