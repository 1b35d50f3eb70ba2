cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python scripts/experiments/exp_pair_rows.py > gpurun_out/r6i_pair.log 2>&1
