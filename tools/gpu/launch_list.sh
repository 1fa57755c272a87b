# ncu launch list (per-kernel durations, serialised) of one default bench step: usage launch_list.sh TAG
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$1.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-shots 65536 \
  > gpurun_out/launches_$1.log 2>&1; echo launches=$?
