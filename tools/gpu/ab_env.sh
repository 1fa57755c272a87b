# A/B of library builds x environment settings: usage ab_env.sh MODEL SHOTS "ENV1" "ENV2" ...
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
model=$1; shots=$2; shift 2
for d in paper_2604_01059_b200/_lib/ab_*/; do
  n=$(basename $d)
  for e in "$@"; do
    env $e ZXS_B200_LIB=$d/libzxs_b200.so timeout 600 python tools/gpu/load_big.py $model $shots $shots > gpurun_out/r2_abe_$n.log 2>&1
    echo "$n $e"; grep "shots $shots" gpurun_out/r2_abe_$n.log | tail -1 | cut -c1-330
  done
done
