cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "dedup or mono or kernel_timing or cultivation" > gpurun_out/pytest36.log 2>&1; echo pytest=$?
tail -4 gpurun_out/pytest36.log
M=data/c3_cultivation_proxy.zxs.gz
for L in ab_head ab_nofold; do
ZXS_DEDUP=0 ZXS_B200_LIB=paper_2604_01059_b200/_lib/$L/libzxs_b200.so timeout 300 python tools/gpu/time_shot.py --model $M --shots $((148*24576)) --reps 3 --tag $L >> gpurun_out/ab36.jsonl 2>>gpurun_out/ab36.err
done
ZXS_DEDUP=0 timeout 300 python tools/gpu/time_shot.py --model $M --shots $((148*24576)) --reps 3 --tag fold >> gpurun_out/ab36.jsonl 2>>gpurun_out/ab36.err
for sh in 1048576 4194304 16777216 67108864; do
ZXS_DEDUP=1 timeout 300 python tools/gpu/time_shot.py --model $M --shots $sh --reps 5 --tag dedup_$sh >> gpurun_out/ab36.jsonl 2>>gpurun_out/ab36.err
done
python -c "
import json
for l in open('gpurun_out/ab36.jsonl'):
    d=json.loads(l); print(d['tag'], d['shots'], '%.2f ms'%d['ms'], '%.4g shots/s'%d['shots_per_s'])"
tail -3 gpurun_out/ab36.err
