# A/B of library builds (paper_2604_01059_b200/_lib/ab_*/) on config 3, 2^28 shots
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for d in paper_2604_01059_b200/_lib/ab_*/; do
  n=$(basename $d)
  ZXS_B200_LIB=$d/libzxs_b200.so timeout 600 python tools/gpu/load_big.py data/c3_cultivation_d3.zxs.xz 268435456 268435456 > gpurun_out/r2_ab_$n.log 2>&1
  echo "$n"; grep "shots 268435456" gpurun_out/r2_ab_$n.log | tail -1 | cut -c1-330
done
