cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc $?"
TMD_TRACE_REBUILD=3 timeout 300 torchrun --standalone --nproc-per-node 2 bench.py --gpus 2 --no-e2e > gpurun_out/bench2_t.log 2>&1
TMD_TRACE_REBUILD=3 timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench1_t.log 2>&1
