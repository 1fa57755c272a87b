set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:shot_kernel -s 2 -c 1 -o gpurun_out/prof_shot_c2_19 python tools/gpu/profile_shot.py --shots 16777216 --launches 3 > gpurun_out/ncu19.log 2>&1; echo ncu=$?
tail -2 gpurun_out/ncu19.log
# torchrun smoke of the multi-GPU code path (1 rank, NCCL)
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench19_torchrun.json 2> gpurun_out/bench19_torchrun.err; echo torchrun=$?; cat gpurun_out/bench19_torchrun.json; tail -3 gpurun_out/bench19_torchrun.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench19_ref.json 2> gpurun_out/bench19_ref.err; echo ref=$?; cat gpurun_out/bench19_ref.json
