cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "multi_gpu" > gpurun_out/pytest_mgpu.log 2>&1
echo "rc $?"
