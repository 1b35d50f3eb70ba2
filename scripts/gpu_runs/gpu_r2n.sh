cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python scripts/experiments/exp_phases.py 80 61,79 > gpurun_out/r2n_exp_phases.log 2>&1
