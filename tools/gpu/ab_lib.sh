# A/B of library builds (paper_2604_01059_b200/_lib/ab_*/): usage ab_lib.sh MODEL SHOTS
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
model=${1:-data/c3_cultivation_d3.zxs.xz}; shots=${2:-268435456}
for d in paper_2604_01059_b200/_lib/ab_*/; do
  n=$(basename $d)
  ZXS_B200_LIB=$d/libzxs_b200.so timeout 600 python tools/gpu/load_big.py $model $shots $shots > gpurun_out/r2_ab_$n.log 2>&1
  echo "$n"; grep "shots $shots" gpurun_out/r2_ab_$n.log | tail -1 | cut -c1-330
done
