cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 torchrun --standalone --nproc-per-node 2 scripts/mgpu_check.py > gpurun_out/mgpu2.log 2>&1
echo "mgpu2 rc $?"
timeout 600 torchrun --standalone --nproc-per-node 4 scripts/mgpu_check.py > gpurun_out/mgpu4.log 2>&1
echo "mgpu4 rc $?"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc $?"
