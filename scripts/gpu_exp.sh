cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc $?"
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench1.log 2>&1
echo "bench1 rc $?"
timeout 600 python scripts/diag_steps.py 80 45 > gpurun_out/diag_steps.log 2>&1
echo "diag rc $?"
