set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for m in c1_surface_d3_zmem c2_surface_d3_xmem_t c4_color_d5_rz3 c5_surface_d7_r7; do
  for S in 2 4; do
    ZXS_SHOTS_PER_LANE=$S timeout 300 python tools/gpu/time_shot.py --model tests/golden/$m.zxs --shots $((148*65536*2)) --reps 7 --tag S$S >> gpurun_out/spl32.jsonl 2>>gpurun_out/spl32.err
  done
done
cat gpurun_out/spl32.jsonl | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['tag'], d['model'].split('/')[-1], '%.4g'%d['shots_per_s'])"
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu32.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu32.log
