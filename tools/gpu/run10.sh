set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -k "mono" > gpurun_out/pytest_mono10.log 2>&1; echo pytest_mono=$?
tail -30 gpurun_out/pytest_mono10.log
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu10.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu10.log
