set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -x -k "dedup or mono or kernel_timing or cultivation" > gpurun_out/pytest34.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest34.log
for D in 1 0; do
ZXS_DEDUP=$D timeout 300 python tools/gpu/time_shot.py --model data/c3_cultivation_proxy.zxs.gz --shots $((148*24576)) --reps 3 --tag dedup$D >> gpurun_out/dedup34.jsonl 2>>gpurun_out/dedup34.err
done
ZXS_DEDUP=1 timeout 300 python tools/gpu/time_shot.py --model data/c3_cultivation_proxy.zxs.gz --shots $((1<<26)) --reps 3 --tag dedup1_64M >> gpurun_out/dedup34.jsonl 2>>gpurun_out/dedup34.err
cat gpurun_out/dedup34.jsonl; tail -5 gpurun_out/dedup34.err
