cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc $?"
for i in 1 2 3 4 5; do
TMD_TRACE_REBUILD=3 timeout 300 torchrun --standalone --nproc-per-node 4 bench.py --gpus 4 --no-e2e > gpurun_out/bench4_$i.log 2>&1
echo "bench4 rc $?"
done
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench1.log 2>&1
