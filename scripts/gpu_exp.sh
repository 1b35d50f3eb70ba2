cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python scripts/experiments/exp_force.py 80 > gpurun_out/exp_force.log 2>&1
echo done
