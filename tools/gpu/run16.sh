set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -k "mono or cultivation" > gpurun_out/pytest_mono16.log 2>&1; echo pytest=$?
tail -4 gpurun_out/pytest_mono16.log
for nw in 1 2; do
ZXS_MONO_WORDS=$nw timeout 300 python tools/gpu/time_shot.py --model tests/golden/surface_d3_xmem_9t.zxs --shots 2424832 --reps 3 --tag 9t_mono_v8_nw$nw 2>&1 | tee -a gpurun_out/t16.json
ZXS_MONO_WORDS=$nw timeout 600 python tools/gpu/time_shot.py --model data/c3_cultivation_proxy.zxs.gz --shots 2424832 --reps 3 --tag cult_mono_v8_nw$nw 2>&1 | tee -a gpurun_out/t16.json
done
ZXS_MONO_WORDS=1 timeout 900 python -m pytest tests -m gpu -q --timeout 600 -k "mono or cultivation" > gpurun_out/pytest_mono16_nw1.log 2>&1; echo pytest_nw1=$?
tail -2 gpurun_out/pytest_mono16_nw1.log
