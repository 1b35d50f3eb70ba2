cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc $?"
timeout 600 torchrun --standalone --nproc-per-node 2 scripts/mgpu_check.py > gpurun_out/mgpu2.log 2>&1
echo "mgpu2 rc $?"
timeout 300 torchrun --standalone --nproc-per-node 2 bench.py --gpus 2 --no-e2e > gpurun_out/bench2.log 2>&1
timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench1.log 2>&1
