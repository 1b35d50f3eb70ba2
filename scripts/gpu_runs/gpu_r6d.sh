cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python scripts/experiments/exp_sorted_rows.py > gpurun_out/r6d_sorted.log 2>&1
