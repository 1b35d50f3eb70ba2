cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc $?"
TMD_TRACE_REBUILD=1 timeout 600 python scripts/mgpu_phases.py 80 100 > gpurun_out/phases1t.log 2>&1
echo "phases rc $?"
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench1.log 2>&1
echo "bench1 rc $?"
