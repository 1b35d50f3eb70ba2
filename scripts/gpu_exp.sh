cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python scripts/experiments/exp_force.py 80 > gpurun_out/exp_force.log 2>&1
TMD_STEP_MINB=6 timeout 600 python scripts/experiments/exp_force.py 80 > gpurun_out/exp_force6.log 2>&1
TMD_STEP_MINB=8 timeout 600 python scripts/experiments/exp_force.py 80 > gpurun_out/exp_force8.log 2>&1
echo done
