cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc $?"
timeout 600 python scripts/experiments/exp_force.py 80 > gpurun_out/exp_force.log 2>&1
for i in 1 2; do
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench1_$i.log 2>&1
done
